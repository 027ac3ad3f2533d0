#!/bin/bash
# compute-sanitizer over the smoke path (one tool per call: TOOL=memcheck|racecheck|synccheck)
TOOL=${TOOL:-memcheck}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_plain_$TOOL.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1200 compute-sanitizer --tool $TOOL --print-limit 50 --error-exitcode 9 \
   python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_$TOOL.log 2>&1
echo "sanitizer rc=$?" >> gpurun_out/sanitizer_$TOOL.log
tail -5 gpurun_out/sanitizer_$TOOL.log
