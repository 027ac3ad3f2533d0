#!/bin/bash
# A/B of library switches on the headline bench line (config 3 only).
#   SETTINGS="label:VAR=value ..." bash tools/ab_bench.sh
for i in 1 2; do
  for s in ${SETTINGS:-default:}; do
    lab=${s%%:*}; kv=${s#*:}
    env $kv python bench.py --steps 30 --warmup 5 --no-extra-configs --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$lab', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), d['stages_ms'])"
  done
done
