#!/bin/bash
OUT=gpurun_out/b8; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solver.py -q -x > $OUT/tests.log 2>&1; tail -3 $OUT/tests.log
timeout 1500 python scripts/ab_matvec.py "sf=0" "sf=1" --rounds 3 > $OUT/ab_sf.txt 2>&1; cat $OUT/ab_sf.txt
