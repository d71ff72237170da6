# A/B: loads batched ahead of the in-order arithmetic in k_segment_sum_gather (GVT_SEG_U entries per lane) and
# k_cg_combine_ap (GVT_CA_U elements per thread) vs one element at a time (ab/libhead.so = before); variants
# seg4 (SEG_U 4, 8 blocks/SM), ca2 (CA_U 2), ca4free (CA_U 4, no register cap)
python -m pytest tests/test_gpu_round2_paths.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "cg_tail or c4_multiterm or symmetric_gemv or medium" 2>&1 | tail -2
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
    np.save(sys.argv[1], a.cpu().numpy())
PY
for k in ranking poly2d linear; do
  GVT_LIBRARY=ab/libhead.so python /tmp/fit10.py /tmp/old_$k.npy $k && python /tmp/fit10.py /tmp/new_$k.npy $k && \
    python -c "import numpy as np; print('bit-identical C4 $k 10-iteration fit:', np.array_equal(np.load('/tmp/old_$k.npy'), np.load('/tmp/new_$k.npy')))"
done
for r in 1 2; do
  for lib in ab/libhead.so paper_2009_01054_b200/libgvt.so ab/libseg4.so ab/libca2.so ab/libca4free.so; do
    echo "$lib $(GVT_LIBRARY=$lib timeout 300 python scripts/fit_probe.py C4 ranking 40 3)"
  done
done
for lib in ab/libhead.so paper_2009_01054_b200/libgvt.so; do
  echo "$lib $(GVT_LIBRARY=$lib timeout 300 python scripts/fit_probe.py C4 poly2d 20 2)"
done
for lib in ab/libhead.so paper_2009_01054_b200/libgvt.so; do
  echo "== $lib (warm cache)"
  GVT_LIBRARY=$lib timeout 600 ncu --clock-control none --cache-control none --kernel-name regex:"segment_sum_gather|combine_ap" -c 6 \
    --metrics gpu__time_duration.sum python scripts/fit_probe.py C4 ranking 6 1 2>&1 | grep -E "k_|duration" | head -12
done
