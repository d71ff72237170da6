# A/B of the longest-K-list-first tile order for the block-sparse stage-1 GEMM (GVT_KBLOCK_ORDER=0: grouped order):
# C4 MLPK parity, slopes, stage-1 phase stamps
python -m pytest tests/test_gpu_parity.py tests/test_gpu_round2_paths.py -x -q -p no:cacheprovider -k "mlpk or c4 or kblock" 2>&1 | tail -2
for rep in 1 2; do for o in 0 1; do
  echo "order=$o $(GVT_KBLOCK_ORDER=$o timeout 300 python scripts/fit_probe.py C4 mlpk 10 2)"
done; done
for o in 0 1; do
  echo "order=$o $(GVT_KBLOCK_ORDER=$o GVT_PROBE_OPTS=OPT_PROFILE=1 GVT_GEMM_PROF=1 timeout 300 python scripts/fit_probe.py C4 mlpk 2 1 2>&1 | grep 'epi=3' | tail -1)"
done
