#!/bin/bash
# One ncu --set full capture of one kernel launch, summaries only.
#   tools/ncu_kernel.sh TAG REGEX SKIP -- command...
TAG=$1; RE=$2; SKIP=$3; shift 4
ncu --set full --clock-control none --import-source on -k regex:$RE -s $SKIP -c 1 \
    -o /tmp/$TAG "$@" > /tmp/ncu_$TAG.log 2>&1
tail -1 /tmp/ncu_$TAG.log
ncu -i /tmp/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
ncu -i /tmp/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/$TAG.ncu-rep --page source --csv > gpurun_out/${TAG}_source.csv 2>/dev/null
