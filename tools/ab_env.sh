#!/bin/bash
# A/B of library switches on one box: spectral step of configs 3, 4, 1 per setting.
#   SETTINGS="base:X=0 new:X=1" bash tools/ab_env.sh      (label:VAR=value, VAR=value optional)
for i in 1 2; do
  for s in ${SETTINGS:-default:}; do
    lab=${s%%:*}; kv=${s#*:}
    for c in ${CONFIGS:-3 4 1}; do env $kv python tools/spectral_bench.py $lab $c; done
  done
done
if [ -n "${TESTS:-}" ]; then
  timeout 900 python -m pytest $TESTS -q 2>&1 | tail -3
fi
