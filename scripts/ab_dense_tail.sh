# A/B of the fused dense-engine CG tail (GVT_DENSE_TAIL=0: separate kernels): its tests, then C3 per-iteration
# slopes (graph-replayed fits, scripts/fit_probe.py) and the tail's phase stamps (eager, GVT_TAIL_PROF)
python -m pytest tests/test_gpu_round2_paths.py -x -q -p no:cacheprovider -k "dense_cg_tail" 2>&1 | tail -5
for k in symmetric antisymmetric kronecker; do
for rep in 1 2; do
GVT_DENSE_TAIL=0 timeout 300 python scripts/fit_probe.py C3 $k 20 3
timeout 300 python scripts/fit_probe.py C3 $k 20 3
done; done
GVT_TAIL_PROF=1 GVT_PROBE_OPTS=OPT_GRAPHS=0 timeout 300 python scripts/fit_probe.py C3 symmetric 6 1 2>&1 | tail -4
