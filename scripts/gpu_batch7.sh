#!/bin/bash
OUT=gpurun_out/b7; mkdir -p $OUT
timeout 900 ncu --set full --import-source on -k regex:k_build_x16 --launch-skip 1 -c 1 -o $OUT/bx16 python scripts/c5_fit_probe.py 2 > $OUT/bx16.log 2>&1
ls -la $OUT
