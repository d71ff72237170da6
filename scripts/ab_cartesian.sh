# The Cartesian kernel's forms on C3: tensor-core D X + X T sampled GEMMs with the fused CG tail (the auto
# choice), the same GEMMs with the separate CG kernels (GVT_DENSE_TAIL=0), and the gather form (OPT_ENGINE=1):
# tests, then per-iteration slopes of graph-replayed fits (scripts/fit_probe.py)
python -m pytest tests/test_gpu_round2_paths.py -x -q -p no:cacheprovider -k "cartesian or dense_cg_tail" 2>&1 | tail -3
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "c3_homogeneous or tiny_vs_explicit or launch_acc" 2>&1 | tail -3
for rep in 1 2; do
GVT_PROBE_OPTS=OPT_ENGINE=1 timeout 300 python scripts/fit_probe.py C3 cartesian 20 3
GVT_DENSE_TAIL=0 timeout 300 python scripts/fit_probe.py C3 cartesian 20 3
timeout 300 python scripts/fit_probe.py C3 cartesian 20 3
done
