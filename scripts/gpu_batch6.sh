#!/bin/bash
OUT=gpurun_out/b6; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_features.py -q -x > $OUT/parity.log 2>&1; tail -3 $OUT/parity.log
timeout 1500 python scripts/ab_matvec.py "ts=1" "ts=0" --rounds 3 > $OUT/ab_ts.txt 2>&1; cat $OUT/ab_ts.txt
