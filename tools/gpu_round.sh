#!/bin/bash
# One GPU call: full -m gpu suite, the multi-body timings, then the default bench line.
set -u
TAG=${1:-run}
python -m pytest tests -m gpu -q > gpurun_out/gputests_$TAG.log 2>&1
echo "tests rc=$?" >> gpurun_out/gputests_$TAG.log
tail -3 gpurun_out/gputests_$TAG.log
python tools/bench_sim.py > gpurun_out/bench_sim_$TAG.log 2>&1; cat gpurun_out/bench_sim_$TAG.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"
tail -c 600 gpurun_out/bench_$TAG.err
