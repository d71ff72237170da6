# A/B of the stage-2 serve's index prefetch (-DSERVE_PREFETCH=0/1 builds under ab/): C4 Poly2D stage-2 phase stamps and
# slopes, C5 fit10; then the C3/C4 parity tests on the default build
for rep in 1 2; do for v in pf0 pf1; do
  echo "$v $(GVT_LIBRARY=ab/lib$v.so GVT_PROBE_OPTS=OPT_PROFILE=1 GVT_GEMM_PROF=1 timeout 300 python scripts/fit_probe.py C4 poly2d 2 1 2>&1 | grep "epi=1" | tail -1)"
  echo "$v $(GVT_LIBRARY=ab/lib$v.so timeout 300 python scripts/fit_probe.py C4 poly2d 10 2)"
  echo "$v $(GVT_LIBRARY=ab/lib$v.so timeout 300 python scripts/fit_probe.py C4 mlpk 10 2)"
done; done
python scripts/ab_matvec.py "lib=ab/libpf0.so" "lib=ab/libpf1.so" --rounds 2
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "c3 or c4 or c5 or tiny" 2>&1 | tail -2
