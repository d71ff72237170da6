"""Probe: error of the tcgen05 3xTF32 Gram vs the fp64 oracle (diagnostics only)."""
import numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O, paper_2009_01054_b200 as G
ctx = G.Context(0)
rng = np.random.default_rng(0)
for m, dim in [(517, 128), (2000, 128), (300, 37)]:
    X = rng.standard_normal((m, dim)).astype(np.float32)
    for kind in (G.BASE_LINEAR, G.BASE_GAUSSIAN):
        ref = O.gram(kind, X, gamma=1.0 / dim)
        for eng, prec in ((1, 0), (2, 0), (2, 1)):
            ctx.set_option(G.OPT_GRAM_ENGINE, eng)
            ctx.set_option(G.OPT_TC_PRECISION, prec)
            K = ctx.gram(kind, torch.from_numpy(X).cuda(), gamma=1.0 / dim).cpu().numpy()
            err = np.abs(K - ref)
            print(f"m={m} dim={dim} kind={kind} engine={'simt' if eng==1 else ('tc-fp16x3' if prec==0 else 'tc-tf32x3')} maxerr={err.max():.3e} "
                  f"rel_to_max={err.max()/np.abs(ref).max():.3e} diag_err={np.abs(np.diag(K)-np.diag(ref)).max():.3e} "
                  f"mean_signed_diag={np.mean(np.diag(K)-np.diag(ref)):.3e}")
