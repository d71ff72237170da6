#!/bin/bash
OUT=gpurun_out/b3; mkdir -p $OUT
timeout 1500 python scripts/ab_matvec.py "gm=16" "gm=8" "gm=4" "gm=32" "gm=2" --rounds 2 > $OUT/ab_gm.txt 2>&1
cat $OUT/ab_gm.txt
for gm in 16 8 4; do
  GVT_GROUP_M=$gm timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k_gemm2_x3 --launch-skip 2 -c 2 --csv python scripts/c5_fit_probe.py 2 > $OUT/ncu_gm$gm.csv 2>&1
  grep -E "dram__bytes_read|gpu__time|hit_rate|per_second" $OUT/ncu_gm$gm.csv | cut -c1-220
done
