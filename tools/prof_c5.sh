#!/bin/bash
# Config-5 slab kernels: launch list, then one ncu --set full capture per kernel
# kind (summaries only: details + raw + source CSVs).   tools/prof_c5.sh TAG
T=${1:-r02}
ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv \
    --log-file gpurun_out/launches_c5_$T.csv python tools/prof_c5.py 3 > /dev/null 2>&1
for k in k_slab_rows_4s k_slab_colsA k_slab_colsB k_slab_evolve; do
  bash tools/ncu_kernel.sh ${k#k_slab_}_c5_$T $k 1 -- python tools/prof_c5.py 3
done
