# A/B: symmetric-GEMV off-diagonal fast path (default) vs the generic masked loop for every unit
# (ab/liboffdiag0.so, -DGVT_SYMV_OFFDIAG=0): bit identity of C4 fits, oracle tests, slopes, ncu
python -m pytest tests/test_gpu_symv.py tests/test_gpu_round2_paths.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "symv or symmetric_gemv or c4_multiterm or cg_tail" 2>&1 | tail -2
cat > /tmp/fit10.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import synth, paper_2009_01054_b200 as G
kname = sys.argv[2]
w = synth.config4()
kernel = getattr(G, kname.upper())
if kernel in G.HOMOGENEOUS_KERNELS: w = synth.union_domain(w)
d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
with G.Context(0) as ctx:
    D = ctx.gram(w.base, d(w.Xd), gamma=w.gamma)
    T = None if w.Xt is None else ctx.gram(w.base, d(w.Xt), gamma=w.gamma)
    a, it, hist, code = ctx.fit(D, T, d(w.train_first), d(w.train_second), d(w.y), G.gvt_kernel_terms(kernel), w.lam, 10)
    st = ctx.stats()
    np.save(sys.argv[1], a.cpu().numpy())
    print(kname, "gemv launches:", st["kinds"]["gemv"]["count"])
PY
for k in ranking mlpk; do
  GVT_LIBRARY=ab/liboffdiag0.so python /tmp/fit10.py /tmp/old_$k.npy $k && python /tmp/fit10.py /tmp/new_$k.npy $k && \
    python -c "import numpy as np; print('bit-identical C4 $k 10-iteration fit:', np.array_equal(np.load('/tmp/old_$k.npy'), np.load('/tmp/new_$k.npy')))"
done
for r in 1 2 3; do
  echo "generic  $(GVT_LIBRARY=ab/liboffdiag0.so timeout 300 python scripts/fit_probe.py C4 ranking 40 3)"
  echo "offdiag  $(timeout 300 python scripts/fit_probe.py C4 ranking 40 3)"
done
for lib in ab/liboffdiag0.so paper_2009_01054_b200/libgvt.so; do
  echo "== $lib (warm cache)"
  GVT_LIBRARY=$lib timeout 600 ncu --clock-control none --cache-control none --kernel-name regex:symv_panel -c 3 \
    --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.sum python scripts/fit_probe.py C4 ranking 4 1 2>&1 | grep -E "duration|dram|inst" | head -9
done
