#!/bin/bash
# Per-config bench lines (C1-C4 and every kernel each config runs), graphs on (--no-profile) and
# a profiled (eager, per-kernel events) pass.  usage: gpurun -- bash scripts/bench_configs.sh TAG
TAG=${1:-cfg}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for wk in "C1 kronecker" "C2 kronecker" "C3 symmetric" "C3 antisymmetric" "C3 cartesian" "C4 poly2d" "C4 mlpk" "C4 ranking"; do
  set -- $wk
  timeout 900 python bench.py --workload $1 --kernel $2 --steps 5 --warmup 3 --no-profile --no-gather-regime >> $OUT/graphs.jsonl 2>> $OUT/err.log
  timeout 600 python bench.py --workload $1 --kernel $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-gather-regime >> $OUT/profiled.jsonl 2>> $OUT/err.log
done
wc -l $OUT/*.jsonl; tail -5 $OUT/err.log
