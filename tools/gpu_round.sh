#!/bin/bash
# One GPU session: parity tests, per-op timings, ncu launch lists + full
# captures per workload, the bench line and the bench's own launch list.
# Everything lands in gpurun_out/ as text; tools/collect_profiles.py turns it
# into profiles/.
#   gpurun --timeout 2400 -- bash tools/gpu_round.sh [workloads...]
set -u
OUT=gpurun_out
mkdir -p $OUT
WS=${*:-c2 c3 c1 c5}
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -3 $OUT/gpu_tests.log
timeout 600 python tools/quick_bench.py $WS > $OUT/quick.log 2>&1; cat $OUT/quick.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"; tail -c 600 $OUT/bench.json
for W in $WS; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file $OUT/launches_$W.csv python tools/profile_ops.py $W > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"compress|decompress|moments|k_add|negate" -c 12 \
      -o /tmp/prof_$W -f python tools/profile_ops.py $W > $OUT/ncu_full_$W.log 2>&1
  ncu -i /tmp/prof_$W.ncu-rep --page raw --csv > $OUT/ncu_raw_$W.csv 2>/dev/null
  ncu -i /tmp/prof_$W.ncu-rep --page details --csv > $OUT/ncu_details_$W.csv 2>/dev/null
  echo "ncu $W done"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_bench.csv python bench.py --steps 2 --warmup 3 > $OUT/bench_under_ncu.log 2>&1
echo "all done"
