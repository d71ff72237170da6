#!/bin/bash
OUT=gpurun_out/b11; mkdir -p $OUT
timeout 1500 python scripts/ab_matvec.py "lib=ab/libX0.so" "lib=ab/libX1.so" --rounds 3 > $OUT/ab_x.txt 2>&1; cat $OUT/ab_x.txt
