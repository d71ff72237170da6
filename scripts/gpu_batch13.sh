#!/bin/bash
OUT=gpurun_out/b13; mkdir -p $OUT
timeout 1500 python scripts/ab_matvec.py "lib=ab/libV0.so" "lib=ab/libV1.so" --rounds 3 > $OUT/ab_v.txt 2>&1; cat $OUT/ab_v.txt
