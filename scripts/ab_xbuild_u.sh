# A/B: entries in flight per lane in the warp-per-row pair-matrix build (-DXB_U=4 default / 8, ab/ builds): C3 slopes
for rep in 1 2; do for k in symmetric cartesian; do for v in xu4 xu8; do
  echo "$v $(GVT_LIBRARY=ab/lib$v.so timeout 300 python scripts/fit_probe.py C3 $k 20 3)"
done; done; done
for v in xu4 xu8; do
  GVT_LIBRARY=ab/lib$v.so GVT_TAIL_PROF=1 GVT_PROBE_OPTS=OPT_GRAPHS=0 timeout 300 python scripts/fit_probe.py C3 symmetric 6 1 2>&1 | grep dense_cg_tail | tail -2
done
