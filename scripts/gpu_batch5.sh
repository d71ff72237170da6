#!/bin/bash
OUT=gpurun_out/b5; mkdir -p $OUT
for wk in C1 C2; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$wk.csv \
  python bench.py --workload $wk --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-profile > $OUT/ncu_$wk.log 2>&1
done
ls -la $OUT
