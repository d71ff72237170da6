#!/bin/bash
# One GPU-box pass: parity tests, smoke, default bench, ncu launch list of the bench command.
# usage (from this container): gpurun --timeout 3000 -- bash scripts/gpu_check.sh [tag]
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $OUT/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
if [ "${NCU:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-gather-regime --no-configs > $OUT/ncu_bench.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_bench.log
fi
tail -3 $OUT/pytest_gpu.log $OUT/smoke.log; cat $OUT/bench.json; tail -3 $OUT/bench.err
