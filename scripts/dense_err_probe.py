"""Probe: sampled matvec error of sparse vs dense engines on C3/C4 kernels (diagnostics)."""
import numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle as O, paper_2009_01054_b200 as G, synth
from test_gpu_parity import sampled_parity
ctx = G.Context(0)
for name, k in [("C3", G.ANTISYMMETRIC), ("C3", G.SYMMETRIC), ("C4u", G.MLPK), ("C4", G.POLY2D)]:
    w = synth.config3() if name == "C3" else synth.config4()
    if name == "C4u": w = synth.union_domain(w)
    for eng, prec in ((1, 0), (2, 0), (2, 1)):
        ctx.set_option(G.OPT_ENGINE, eng)
        ctx.set_option(G.OPT_TC_PRECISION, prec)
        r, u, idx = sampled_parity(ctx, w, k, k_samples=48)
        print(name, k, "sparse" if eng == 1 else ("dense-fp16x3" if prec == 0 else "dense-tf32x3"), f"rel={r:.3e}", flush=True)
