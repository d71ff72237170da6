#!/bin/bash
OUT=gpurun_out/b4; mkdir -p $OUT
timeout 1500 python scripts/ab_matvec.py "lib=ab/libA.so" "lib=ab/libB.so" --rounds 3 > $OUT/ab_stage.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "in_loop" > $OUT/inloop.log 2>&1
cat $OUT/ab_stage.txt; tail -5 $OUT/inloop.log
