#!/bin/bash
OUT=gpurun_out/b13; mkdir -p $OUT
timeout 1500 python scripts/ab_matvec.py "lib=ab/libKC4.so" "lib=ab/libKC8.so" --rounds 3 > $OUT/ab_kc.txt 2>&1; cat $OUT/ab_kc.txt
