#!/bin/bash
# ncu --set full of one op's kernel: tools/prof_one.sh <workload> <op> <kernel-regex>
set -u
W=$1; OP=$2; K=$3
mkdir -p gpurun_out
PROFILE_ONLY=$OP timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -f -o /tmp/p_${W}_$OP python tools/profile_ops.py $W > gpurun_out/ncu_${W}_$OP.log 2>&1
ncu -i /tmp/p_${W}_$OP.ncu-rep --page details --csv > gpurun_out/det_${W}_$OP.csv 2>/dev/null
ncu -i /tmp/p_${W}_$OP.ncu-rep --page raw --csv > gpurun_out/raw_${W}_$OP.csv 2>/dev/null
ncu -i /tmp/p_${W}_$OP.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${W}_$OP.csv 2>/dev/null
