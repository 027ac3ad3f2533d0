#!/bin/bash
# Config-5 slab kernels: time, then one ncu --set full capture per kernel kind
# (summaries only: details + raw + source CSVs).
python tools/prof_c5.py 3 > gpurun_out/c5_plain.log 2>&1 && cat gpurun_out/c5_plain.log
for k in k_slab_rows k_slab_colsA k_slab_colsB; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o /tmp/$k python tools/prof_c5.py 3 > /tmp/ncu_$k.log 2>&1
  tail -1 /tmp/ncu_$k.log
  ncu -i /tmp/$k.ncu-rep --page details --csv > gpurun_out/${k}_details.csv 2>/dev/null
  ncu -i /tmp/$k.ncu-rep --page raw --csv > gpurun_out/${k}_raw.csv 2>/dev/null
  ncu -i /tmp/$k.ncu-rep --page source --csv > gpurun_out/${k}_source.csv 2>/dev/null
done
# config-3 row pass (second velocity group: grids 2-3)
ncu --set full --clock-control none --import-source on -k regex:k_rows_w -s 5 -c 1 \
    -o /tmp/rows3 python tools/spectral_bench.py rows > /tmp/ncu_rows3.log 2>&1
tail -1 /tmp/ncu_rows3.log
ncu -i /tmp/rows3.ncu-rep --page details --csv > gpurun_out/rows3_details.csv 2>/dev/null
ncu -i /tmp/rows3.ncu-rep --page raw --csv > gpurun_out/rows3_raw.csv 2>/dev/null
ncu -i /tmp/rows3.ncu-rep --page source --csv > gpurun_out/rows3_source.csv 2>/dev/null
