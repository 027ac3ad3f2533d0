#!/bin/bash
# A/B of column-pass variants on the config-3 spectral step (one box, one build),
# then one ncu capture of the velocity column group per new variant (summaries
# only come back: raw metrics + source-level stall CSVs).
for i in 1 2; do
  python tools/spectral_bench.py tma
  OCN_COLS=direct python tools/spectral_bench.py direct
  OCN_COLS=tma2 python tools/spectral_bench.py tma2
done
OCN_COLS=tma2 python -m pytest tests/test_gpu_benchconfig.py -q -x -k "spectral_step" 2>&1 | tail -2
for v in ${NCU_VARIANTS:-tma direct tma2}; do
  OCN_COLS=$v ncu --set full --clock-control none --import-source on -k regex:k_cols -s 7 -c 1 \
     -o /tmp/cols_$v python tools/spectral_bench.py $v > /tmp/ncu_$v.log 2>&1
  tail -3 /tmp/ncu_$v.log
  ncu -i /tmp/cols_$v.ncu-rep --page raw --csv > gpurun_out/cols_${v}_raw.csv 2>/dev/null
  ncu -i /tmp/cols_$v.ncu-rep --page details --csv > gpurun_out/cols_${v}_details.csv 2>/dev/null
  ncu -i /tmp/cols_$v.ncu-rep --page source --csv > gpurun_out/cols_${v}_source.csv 2>/dev/null
done
du -sh gpurun_out
