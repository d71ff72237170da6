# A/B of the stage-1 (fp16 store) tail split (GVT_STORE_TAIL_SPLIT=0: unsplit): C4 parity tests, C4 slopes, C5 fit10
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "c4 or c5 or predict or slab" 2>&1 | tail -3
for k in poly2d mlpk; do for rep in 1 2; do
  echo "off $(GVT_STORE_TAIL_SPLIT=0 timeout 300 python scripts/fit_probe.py C4 $k 10 2)"
  echo "on  $(timeout 300 python scripts/fit_probe.py C4 $k 10 2)"
done; done
GVT_PROBE_OPTS=OPT_PROFILE=1 GVT_GEMM_PROF=1 timeout 300 python scripts/fit_probe.py C4 poly2d 2 1 2>&1 | grep "epi=3" | tail -1
python scripts/ab_matvec.py "E_GVT_STORE_TAIL_SPLIT=0" "E_GVT_STORE_TAIL_SPLIT=1" --rounds 2
