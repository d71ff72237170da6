#!/bin/bash
OUT=gpurun_out/b13; mkdir -p $OUT
timeout 1500 python scripts/ab_matvec.py "lib=ab/libK0.so" "lib=ab/libK1.so" --rounds 3 > $OUT/ab_k.txt 2>&1; cat $OUT/ab_k.txt
