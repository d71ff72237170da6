# A/B: the persistent small solver stores p_k in phase D by its owner (contiguous) instead of in phase C scattered by
# dst (ab/libsmallold.so = before): C2 per-iteration slopes, phase stamps; the small-engine and S30 tests
python -m pytest tests/test_gpu_solver.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "small or s30 or c2" 2>&1 | tail -2
for r in 1 2 3; do
  echo "old $(GVT_LIBRARY=ab/libsmallold.so timeout 300 python scripts/fit_probe.py C2 kronecker 40 3)"
  echo "new $(timeout 300 python scripts/fit_probe.py C2 kronecker 40 3)"
done
for v in ab/libsmallold.so paper_2009_01054_b200/libgvt.so; do
  GVT_LIBRARY=$v GVT_SMALL_PROF=1 GVT_PROBE_OPTS=OPT_GRAPHS=0 timeout 300 python scripts/fit_probe.py C2 kronecker 10 1 2>&1 | grep small_cg | tail -2
done
