#!/bin/bash
# A/B of column-pass variants (one box, one build): configs 3, 4, 1 spectral steps,
# the spectral parity tests under the new variant, optional ncu captures.
V=${VARIANTS:-tma tmaw}
for i in 1 2; do
  for v in $V; do OCN_COLS=$v python tools/spectral_bench.py $v; done
done
for v in $V; do OCN_COLS=$v python tools/spectral_bench.py $v 4; OCN_COLS=$v python tools/spectral_bench.py $v 1; done
OCN_COLS=${TEST_VARIANT:-tmaw} timeout 900 python -m pytest tests/test_gpu_benchconfig.py tests/test_gpu_spectral.py -q -k "spectral_step or instances or frames or maps or slices or assembly" 2>&1 | tail -3
for v in ${NCU_VARIANTS:-}; do
  OCN_COLS=$v ncu --set full --clock-control none --import-source on -k regex:k_cols -s 7 -c 1 \
     -o /tmp/cols_$v python tools/spectral_bench.py $v > /tmp/ncu_$v.log 2>&1
  tail -1 /tmp/ncu_$v.log
  ncu -i /tmp/cols_$v.ncu-rep --page raw --csv > gpurun_out/cols_${v}_raw.csv 2>/dev/null
  ncu -i /tmp/cols_$v.ncu-rep --page details --csv > gpurun_out/cols_${v}_details.csv 2>/dev/null
  ncu -i /tmp/cols_$v.ncu-rep --page source --csv > gpurun_out/cols_${v}_source.csv 2>/dev/null
done
if [ -n "${FULL_TESTS:-}" ]; then
  python -m pytest tests -m gpu -q > gpurun_out/gputests_ab.log 2>&1; tail -15 gpurun_out/gputests_ab.log
fi
