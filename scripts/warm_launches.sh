#!/bin/bash
# Warm-cache per-kernel durations of a few fit iterations (ncu --cache-control none --clock-control none):
# the kernels of a graph-replayed iteration see warm L2, which the default (flushing) launch list hides.
# usage: gpurun -- bash scripts/warm_launches.sh TAG "C3 symmetric" ["C4 ranking" ...]
TAG=$1; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
for wk in "$@"; do
  set -- $wk
  ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
      --log-file $OUT/warm_$1_$2.csv python scripts/fit_probe.py $1 $2 6 1 > /dev/null 2>&1
  python scripts/summarize_ncu.py tail $OUT/warm_$1_$2.csv 14
done
