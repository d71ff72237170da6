#!/bin/bash
OUT=gpurun_out/b10; mkdir -p $OUT
timeout 1500 python scripts/ab_matvec.py "lib=ab/libU1.so" "lib=ab/libU2.so" "lib=ab/libU4.so" --rounds 2 > $OUT/ab_u.txt 2>&1; cat $OUT/ab_u.txt
for U in 1 2 4; do echo "U=$U"; GVT_LIBRARY=ab/libU$U.so python scripts/iter_cost.py C2 C3 2>&1 | tail -2; done
