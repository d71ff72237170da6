# A/B: CTAs per SM of the fused dense tail (GVT_TAIL_CTAS_PER_SM cap = 1 / 2 / 3), C3 per-iteration slopes and phase
# stamps; then the tail's bit-identity tests at the default
for rep in 1 2; do for k in symmetric cartesian; do for c in 2 3; do
  echo "ctas/SM=$c $(GVT_TAIL_CTAS_PER_SM=$c timeout 300 python scripts/fit_probe.py C3 $k 20 3)"
done; done; done
for c in 2 3; do
  GVT_TAIL_CTAS_PER_SM=$c GVT_TAIL_PROF=1 GVT_PROBE_OPTS=OPT_GRAPHS=0 timeout 300 python scripts/fit_probe.py C3 symmetric 6 1 2>&1 | grep dense_cg_tail | tail -2
done
python -m pytest tests/test_gpu_round2_paths.py tests/test_gpu_solver.py -x -q -p no:cacheprovider -k "dense" 2>&1 | tail -2
