# C4 Poly2D / MLPK / Ranking per-iteration slopes and a warm launch list of C4 Poly2D (after a kernel change)
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "c4" 2>&1 | tail -2
for rep in 1 2; do for k in poly2d mlpk ranking; do timeout 300 python scripts/fit_probe.py C4 $k 10 2; done; done
bash scripts/warm_launches.sh c4w3 "C4 poly2d"
