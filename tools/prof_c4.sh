#!/bin/bash
# Launch list of config 4 (64 instances x 3 x 512^2) and full captures of its passes.
T=${1:-r02}
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/launches_c4_$T.csv python tools/spectral_bench.py x 4 > /dev/null 2>&1
bash tools/ncu_kernel.sh c4cols_$T k_cols 3 -- python tools/spectral_bench.py x 4
bash tools/ncu_kernel.sh c4rows_$T k_rows 3 -- python tools/spectral_bench.py x 4
bash tools/ncu_kernel.sh c4evo_$T k_evolve 3 -- python tools/spectral_bench.py x 4
