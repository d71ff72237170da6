# A/B: k_symv_finish with every load of a group in flight (16 chunk loads, 8 panel loads) vs four at a time
# (ab/libsymvold.so = before): bit identity of a C4 Ranking fit, per-iteration slopes, warm ncu durations
python -m pytest tests/test_gpu_symv.py tests/test_gpu_round2_paths.py -q -p no:cacheprovider -k "symv or symmetric_gemv" 2>&1 | tail -2
cat > /tmp/symv_fit.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import synth, paper_2009_01054_b200 as G
w = synth.union_domain(synth.config4())
d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
with G.Context(0) as ctx:
    D = ctx.gram(w.base, d(w.Xd), gamma=w.gamma)
    a, it, hist, code = ctx.fit(D, None, d(w.train_first), d(w.train_second), d(w.y), G.gvt_kernel_terms(G.RANKING), w.lam, 10)
    np.save(sys.argv[1], a.cpu().numpy())
PY
GVT_LIBRARY=ab/libsymvold.so python /tmp/symv_fit.py /tmp/old.npy && python /tmp/symv_fit.py /tmp/new.npy && \
  python -c "import numpy as np; print('bit-identical C4 Ranking 10-iteration fit:', np.array_equal(np.load('/tmp/old.npy'), np.load('/tmp/new.npy')))"
for r in 1 2 3; do
  echo "old $(GVT_LIBRARY=ab/libsymvold.so timeout 300 python scripts/fit_probe.py C4 ranking 40 3)"
  echo "new $(timeout 300 python scripts/fit_probe.py C4 ranking 40 3)"
done
for lib in ab/libsymvold.so paper_2009_01054_b200/libgvt.so; do
  echo "== $lib (warm cache)"
  GVT_LIBRARY=$lib timeout 600 ncu --clock-control none --cache-control none --kernel-name regex:symv -c 8 \
    --metrics gpu__time_duration.sum python scripts/fit_probe.py C4 ranking 6 1 2>&1 | grep -E "duration" | head -8
done
