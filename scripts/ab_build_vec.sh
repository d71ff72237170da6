# A/B: 4 cells per thread per pass in the shared-memory sweeps (zero, max, store) of the CTA-per-row
# pair-matrix build (GVT_BUILD_VEC=1 default / 0): C5 bench kernel_ms.densify and step, C4 slopes
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-gather-regime --no-configs"
for rep in 1 2; do for v in 0 1; do
  echo "vec=$v $(GVT_BUILD_VEC=$v timeout 600 $B 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('ms_per_step', round(d['ms_per_step'],1), 'densify_ms', d['kernel_ms'].get('densify'), 'sm_mhz', d['clocks']['sm_mhz'])")"
done; done
for rep in 1 2; do for k in poly2d mlpk; do for v in 0 1; do
  echo "vec=$v $(GVT_BUILD_VEC=$v timeout 300 python scripts/fit_probe.py C4 $k 20 3)"
done; done; done
