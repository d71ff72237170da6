# A/B of the tail split of the sampled GEMM's last partial wave (GVT_TAIL_SPLIT=0: unsplit): C4 parity tests,
# then per-iteration slopes (scripts/fit_probe.py) and the stage-2 phase stamps (GVT_GEMM_PROF)
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "c4 or predict" 2>&1 | tail -3
for k in poly2d mlpk; do for rep in 1 2; do
  echo "off $(GVT_TAIL_SPLIT=0 timeout 300 python scripts/fit_probe.py C4 $k 10 2)"
  echo "on  $(timeout 300 python scripts/fit_probe.py C4 $k 10 2)"
done; done
GVT_PROBE_OPTS=OPT_PROFILE=1 GVT_GEMM_PROF=1 timeout 300 python scripts/fit_probe.py C4 poly2d 2 1 2>&1 | grep "epi=1" | tail -2
