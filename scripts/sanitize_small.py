"""Small end-to-end exercise of every kernel family for compute-sanitizer runs."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01054_b200 as G, synth

ctx = G.Context(0)
d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
rng = np.random.default_rng(0)
for hom in (False, True):
    m, q = 300, (300 if hom else 170)
    D = ctx.gram(G.BASE_GAUSSIAN, d(rng.standard_normal((m, 9)).astype(np.float32)), gamma=0.2)
    T = None if hom else ctx.gram(G.BASE_LINEAR, d(rng.standard_normal((q, 9)).astype(np.float32)))
    f, s = d(rng.integers(0, m, 7001).astype(np.int32)), d(rng.integers(0, q, 7001).astype(np.int32))
    of, os_ = d(rng.integers(0, m, 999).astype(np.int32)), d(rng.integers(0, q, 999).astype(np.int32))
    y = d(rng.standard_normal(7001).astype(np.float32))
    kernels = [G.SYMMETRIC, G.ANTISYMMETRIC, G.RANKING, G.MLPK] if hom else [G.LINEAR, G.POLY2D, G.KRONECKER, G.CARTESIAN]
    for eng, cta, slabs in ((1, 2, 1), (2, 2, 1), (2, 1, 1), (2, 2, 3)):
        ctx.set_option(G.OPT_ENGINE, eng); ctx.set_option(G.OPT_GEMM_CTA, cta); ctx.set_option(G.OPT_SLABS, slabs)
        for k in kernels:
            t = G.gvt_kernel_terms(k)
            a, it, _, _ = ctx.fit(D, T, f, s, y, t, 1.0, 3)
            u = ctx.predict(D, T, of, os_, f, s, a, t)
            torch.cuda.synchronize()
    print("hom", hom, "ok")
print("sanitize_small done")
