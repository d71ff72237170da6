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

# ---- solver / early stopping / AUC / novel objects / Tanimoto (session-2 additions)
rng = np.random.default_rng(1)
m, q = 37, 29
Xd, Xt = rng.standard_normal((m, 5)).astype(np.float32), rng.standard_normal((q, 5)).astype(np.float32)
D = ctx.gram(G.BASE_GAUSSIAN, d(Xd), gamma=0.3)
T = ctx.gram(G.BASE_GAUSSIAN, d(Xt), gamma=0.3)
f, s = d(rng.integers(0, m, 301).astype(np.int32)), d(rng.integers(0, q, 301).astype(np.int32))
y = d(rng.standard_normal(301).astype(np.float32))
vf, vs = d(rng.integers(0, m, 77).astype(np.int32)), d(rng.integers(0, q, 77).astype(np.int32))
vl = d((rng.uniform(size=77) > 0.5).astype(np.float32))
kron = G.gvt_kernel_terms(G.KRONECKER)
for eng in (1, 2):
    ctx.set_option(G.OPT_ENGINE, eng); ctx.set_option(G.OPT_SLABS, 1)
    for solver in (0, 1):
        ctx.set_option(G.OPT_SOLVER, solver)
        ctx.fit(D, T, f, s, y, kron, 0.5, 7)
        ctx.fit(D, T, f, s, y, kron, 0.5, 40, 1e-3)
        ctx.fit_early_stopping(D, T, f, s, y, vf, vs, vl, kron, 0.5, 3, 9)
    ctx.set_option(G.OPT_SOLVER, 0)
    print("auc", ctx.auc(vl, d(rng.standard_normal(77).astype(np.float32))))
    Xn = rng.standard_normal((11, 5)).astype(np.float32)
    Dx = ctx.gram_cross(G.BASE_GAUSSIAN, d(Xn), d(Xd), gamma=0.3)
    Tx = ctx.gram_cross(G.BASE_GAUSSIAN, d(Xt[:13]), d(Xt), gamma=0.3)
    tf, ts = d(rng.integers(0, 11, 55).astype(np.int32)), d(rng.integers(0, 13, 55).astype(np.int32))
    for var in (0, 1, 2):
        ctx.matvec_rect(Dx, Tx, tf, ts, f, s, y, kron, variant=var)
    Dh = ctx.gram_cross(G.BASE_GAUSSIAN, d(Xn), d(Xd), gamma=0.3)
    hf, hs = d(rng.integers(0, m, 301).astype(np.int32)), d(rng.integers(0, m, 301).astype(np.int32))
    for k in (G.SYMMETRIC, G.MLPK, G.POLY2D, G.RANKING):
        terms = G.gvt_kernel_terms(k)
        if k == G.POLY2D:
            ctx.matvec_rect(Dx, Tx, tf, ts, f, s, y, terms)
        else:
            ctx.matvec_rect(Dh, None, tf, d(rng.integers(0, 11, 55).astype(np.int32)), hf, hs, y, terms)
B = (rng.uniform(size=(70, 300)) < 0.1).astype(np.float32)
ctx.gram(G.BASE_TANIMOTO, d(B))
ctx.gram_cross(G.BASE_TANIMOTO, d(B), d(B[:33]))
torch.cuda.synchronize()
print("sanitize_small additions done")

# ---- round-2 paths: symmetric GEMV (square Gram >= 6144), fused CG tail (Ranking / Linear / Poly2D),
#      split-K sampled GEMM and single-unit epilogues (few pair tiles, K >= 1024), warp-per-row X build
rng = np.random.default_rng(2)
ctx2 = G.Context(0)
m = 6200
Dn = ctx2.gram(G.BASE_GAUSSIAN, d(rng.standard_normal((m, 8)).astype(np.float32)), gamma=0.1)
f = d(rng.integers(0, m, 20000).astype(np.int32)); s = d(rng.integers(0, m, 20000).astype(np.int32))
y = d(rng.standard_normal(20000).astype(np.float32))
for k in (G.RANKING, G.LINEAR):
    t = G.gvt_kernel_terms(k)
    a, _, _, _ = ctx2.fit(Dn, None if k == G.RANKING else Dn, f, s, y, t, 1.0, 3)
    torch.cuda.synchronize()
print("symv + cg tail ok")
m = 1100
Dm = ctx2.gram(G.BASE_GAUSSIAN, d(rng.standard_normal((m, 8)).astype(np.float32)), gamma=0.1)
i = rng.integers(0, m, 30000); j = rng.integers(0, m, 30000); keep = i < j
f = d(i[keep].astype(np.int32)); s = d(j[keep].astype(np.int32)); n = int(keep.sum())
y = d(rng.standard_normal(n).astype(np.float32))
ctx2.set_option(G.OPT_ENGINE, 2)
for k in (G.SYMMETRIC, G.KRONECKER):
    t = G.gvt_kernel_terms(k)
    a, _, _, _ = ctx2.fit(Dm, None if k == G.SYMMETRIC else Dm, f, s, y, t, 1.0, 3)
    u = ctx2.matvec(Dm, None if k == G.SYMMETRIC else Dm, f, s, f, s, a, t)
    torch.cuda.synchronize()
print("split-K + single-unit epilogues + warp build ok")
ctx2.close()
