# A/B on the final tree: GEMM rasterization group GROUP_M 16 (default) vs 8 vs 12 -- C5 10-iteration fit times and the
# DRAM bytes of one stage-1 and one stage-2 launch per setting (ncu, dram metrics only)
python scripts/ab_matvec.py "gm=16" "gm=8" "gm=12" --rounds 2 2>&1 | grep round
for gm in 16 8 12; do
  echo "== GVT_GROUP_M=$gm"
  GVT_GROUP_M=$gm timeout 900 ncu --clock-control none -k regex:k_gemm2_x3 --launch-skip 2 -c 2 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct python scripts/c5_fit_once.py 2>&1 | grep -E "k_gemm2|duration|dram|lts"
done
