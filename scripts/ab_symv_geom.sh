# A/B: symmetric-GEMV panel geometry (panel width PW, row chunk RC, rows per batch RB) on C4 Ranking's 8000^2 union
# Gram: matvec agreement with the default build (PW 1024, RC 64, RB 8), per-iteration slopes, ncu durations
cat > /tmp/rk_mv.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import synth, paper_2009_01054_b200 as G
w = synth.union_domain(synth.config4())
d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
with G.Context(0) as ctx:
    D = ctx.gram(w.base, d(w.Xd), gamma=w.gamma)
    f, s = d(w.train_first), d(w.train_second)
    u = ctx.matvec(D, None, f, s, f, s, d(synth.random_vector(3, w.n)), G.gvt_kernel_terms(G.RANKING))
    np.save(sys.argv[1], u.cpu().numpy())
PY
python /tmp/rk_mv.py /tmp/ref.npy
LIBS="paper_2009_01054_b200/libgvt.so ab/libpw2k16.so ab/libpw2k32.so ab/libpw1k32.so ab/libpw1k64rb4.so ab/libpw4k8.so"
for lib in $LIBS; do
  GVT_LIBRARY=$lib python /tmp/rk_mv.py /tmp/x.npy && python -c "
import numpy as np; a=np.load('/tmp/x.npy').astype(np.float64); b=np.load('/tmp/ref.npy').astype(np.float64)
print('$lib rel vs default:', np.linalg.norm(a-b)/np.linalg.norm(b))"
done
for r in 1 2; do for lib in $LIBS; do
  echo "$lib $(GVT_LIBRARY=$lib timeout 300 python scripts/fit_probe.py C4 ranking 40 3)"
done; done
for lib in $LIBS; do
  echo "== $lib (warm cache)"
  GVT_LIBRARY=$lib timeout 600 ncu --clock-control none --cache-control none --kernel-name regex:symv -c 4 \
    --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed python scripts/fit_probe.py C4 ranking 4 1 2>&1 | grep -E "duration|dram" | head -8
done
