#!/bin/bash
# full ncu capture + SASS source page of one kernel in `tools/profile_ops.py <workload>`
# usage: tools/ncu_src.sh <tag> <workload> <kernel-regex> [env...]
set -u
T=$1; W=$2; K=$3; shift 3
mkdir -p gpurun_out
env "$@" ncu --set full --clock-control none --import-source on -k regex:"$K" -c 1 \
    -f -o /tmp/prof_$T python tools/profile_ops.py $W > gpurun_out/ncu_$T.log 2>&1
ncu -i /tmp/prof_$T.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$T.csv 2>/dev/null
ncu -i /tmp/prof_$T.ncu-rep --page details --csv > gpurun_out/ncu_details_$T.csv 2>/dev/null
ncu -i /tmp/prof_$T.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$T.csv 2>/dev/null
