#!/bin/bash
OUT=gpurun_out/b9; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/tests.log 2>&1; tail -2 $OUT/tests.log
bash scripts/bench_configs.sh b9cfg > /dev/null 2>&1
python scripts/iter_cost.py C2 C3 2>&1 | tail -2
