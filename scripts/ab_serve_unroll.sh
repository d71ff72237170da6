# A/B of the stage-2 serve loop's samples in flight per thread (-DSERVE_UNROLL=1/2/4 builds under ab/): C5 fit10
# (scripts/ab_matvec.py) and C4 Poly2D per-iteration slopes
python scripts/ab_matvec.py "lib=ab/libsu1.so" "lib=ab/libsu2.so" "lib=ab/libsu4.so" --rounds 2
for rep in 1 2; do for v in su1 su2 su4; do
  echo "$v $(GVT_LIBRARY=ab/lib$v.so timeout 300 python scripts/fit_probe.py C4 poly2d 10 2)"
done; done
