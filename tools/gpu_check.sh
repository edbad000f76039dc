#!/bin/bash
# Quick GPU round: tests (optionally a -k filter), the default bench line and
# optional extra bench workloads.  usage: tools/gpu_check.sh "<pytest -k expr or ''>" [workloads...]
set -u
OUT=gpurun_out
mkdir -p $OUT
K=${1:-}
shift || true
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -k "$K" > $OUT/gpu_tests.log 2>&1
else
  timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/gpu_tests.log 2>&1
fi
echo "tests rc=$?"; grep -E "passed|failed|error" $OUT/gpu_tests.log | tail -5
grep -E "^(FAILED|ERROR)" $OUT/gpu_tests.log | head -20
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"; tail -c 3000 $OUT/bench.json; tail -5 $OUT/bench.err
for W in "$@"; do
  timeout 900 python bench.py --workload $W --steps 10 > $OUT/bench_$W.json 2> $OUT/bench_$W.err
  echo "bench $W rc=$?"; tail -c 2500 $OUT/bench_$W.json; tail -3 $OUT/bench_$W.err
done
