#!/bin/bash
# one full ncu capture of kernels matching a regex in `tools/profile_ops.py <workload>`
# usage: tools/ncu_one.sh <tag> <workload> <kernel-regex> <count> [env...]
set -u
T=$1; W=$2; K=$3; C=$4; shift 4
mkdir -p gpurun_out
env "$@" ncu --set full --clock-control none --import-source on -k regex:"$K" -c $C \
    -f -o /tmp/prof_$T python tools/profile_ops.py $W > gpurun_out/ncu_$T.log 2>&1
ncu -i /tmp/prof_$T.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$T.csv 2>/dev/null
ncu -i /tmp/prof_$T.ncu-rep --page details --csv > gpurun_out/ncu_details_$T.csv 2>/dev/null
