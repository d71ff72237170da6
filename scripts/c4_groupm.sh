# C4 Poly2D / MLPK per-iteration slope against the CTA-pair GEMM rasterization group (GVT_GROUP_M), then one
# ncu --set full capture of each C4 Poly2D GEMM (DRAM bytes, L2 hit rate, tensor-pipe activity)
for gm in 16 8 4 2 16 8 4 2; do
  echo "GROUP_M=$gm $(GVT_GROUP_M=$gm timeout 300 python scripts/fit_probe.py C4 poly2d 10 2)"
done
for gm in 16 4; do
  echo "GROUP_M=$gm $(GVT_GROUP_M=$gm timeout 300 python scripts/fit_probe.py C4 mlpk 10 2)"
done
ncu --set full --clock-control none -k regex:"k_gemm2_x3" -s 4 -c 2 -o gpurun_out/c4gemm python scripts/fit_probe.py C4 poly2d 2 1 > /dev/null 2>&1
