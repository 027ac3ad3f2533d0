#!/bin/bash
# Round-end evidence for profiles/: launch list of the config-3 frame, the
# spectral kernels' DRAM traffic (application replay, no cache flush), and one
# ncu --set full capture of the merged column launch.   tools/prof_final.sh TAG
T=${1:-r02}
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
    --log-file gpurun_out/launches_frame_$T.csv python tools/prof_frame.py 3 > /dev/null 2>&1
ncu --replay-mode application --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    -k regex:'k_evolve|k_rows_w|k_cols_tma' --csv --log-file gpurun_out/traffic_$T.csv \
    python tools/prof_frame.py 3 > /dev/null 2>&1
# one column launch per frame (merged): the third frame's; row launches 2 per frame
bash tools/ncu_kernel.sh cols_$T k_cols_tma 2 -- python tools/prof_frame.py 3
bash tools/ncu_kernel.sh rowsv_$T k_rows_w 5 -- python tools/prof_frame.py 3
