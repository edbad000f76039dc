#!/bin/bash
# Bench lines of every workload + the per-op quick bench + the default bench's
# ncu launch list (kernel share of the step).  gpurun -- bash tools/gpu_bench_all.sh
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python tools/quick_bench.py c2 c3 c5 c1 > $OUT/quick_all.log 2>&1
for W in c2 c3 c4 c5; do
  timeout 900 python bench.py --workload $W > $OUT/bench_$W.json 2> $OUT/bench_$W.err
  echo "bench $W rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_bench.csv python bench.py --steps 2 --warmup 3 > $OUT/bench_under_ncu.log 2>&1
echo "all done"
