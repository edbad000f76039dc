#!/bin/bash
# ncu evidence for one workload; leaves only text summaries in gpurun_out/.
# usage: tools/ncu_capture.sh <workload> <kernel-regex> <count>
set -u
W=${1:-c2}; K=${2:-"k_"}; C=${3:-6}
OUT=gpurun_out
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/launches_$W.csv python tools/profile_ops.py $W > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"$K" -c $C \
    -o /tmp/prof_$W python tools/profile_ops.py $W > $OUT/ncu_full_$W.log 2>&1
ncu -i /tmp/prof_$W.ncu-rep --page raw --csv > $OUT/ncu_raw_$W.csv 2>/dev/null
ncu -i /tmp/prof_$W.ncu-rep --page details --csv > $OUT/ncu_details_$W.csv 2>/dev/null
ls -la /tmp/prof_$W.ncu-rep >> $OUT/ncu_full_$W.log
