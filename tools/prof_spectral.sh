#!/bin/bash
# Launch list of the config-3 spectral step plus full captures of its column
# and row passes (summaries as CSV into gpurun_out/).   tools/prof_spectral.sh TAG
T=${1:-r02}
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_spectral_$T.csv python tools/spectral_bench.py x 3 > /dev/null 2>&1
bash tools/ncu_kernel.sh cols_$T k_cols 7 -- python tools/spectral_bench.py x 3
bash tools/ncu_kernel.sh rowsw_$T k_rows_w 3 -- python tools/spectral_bench.py x 3
bash tools/ncu_kernel.sh evo_$T k_evolve 3 -- python tools/spectral_bench.py x 3
