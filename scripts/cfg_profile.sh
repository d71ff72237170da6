#!/bin/bash
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "s30 or solver_direction" > $OUT/pytest_s30.log 2>&1; echo "rc=$?" >> $OUT/pytest_s30.log
for wk in "C3 symmetric" "C4 ranking" "C3 cartesian"; do
  set -- $wk
  timeout 600 python bench.py --workload $1 --kernel $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-gather-regime --no-configs >> $OUT/profiled.jsonl 2>> $OUT/err.log
done
tail -3 $OUT/pytest_s30.log
