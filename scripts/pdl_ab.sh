#!/bin/bash
# A/B of programmatic dependent launch (GVT_PDL=1 default vs 0) on the per-iteration cost of the
# latency-bound configs, then the GPU test suite.  usage: gpurun -- bash scripts/pdl_ab.sh TAG
OUT=gpurun_out/$1; mkdir -p $OUT
for r in 0 1; do
for pdl in 0 1; do
for wk in "C2 kronecker" "C3 symmetric" "C3 cartesian" "C4 ranking" "C4 poly2d" "C1 kronecker"; do
  set -- $wk
  echo -n "pdl=$pdl " >> $OUT/pdl_ab.txt
  GVT_PDL=$pdl python scripts/fit_probe.py $1 $2 20 3 >> $OUT/pdl_ab.txt 2>>$OUT/err.log
done; done; done
cat $OUT/pdl_ab.txt
