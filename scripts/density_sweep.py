"""Density dispatch threshold, measured ("Density dispatch threshold (to verify by
measurement)").  At C5 object counts (m = q = 20 000, Gaussian Grams on dim-128 N(0,1) features),
uniform training pairs at a sweep of pair-matrix densities; one training matvec (out = in sample,
plan included) on the sparse SIMT engine and on the dense tensor-core engine, median of 3 after a
warm-up, plus what the auto engine picks.  usage: python scripts/density_sweep.py [--m M]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01054_b200 as G  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=20_000)
ap.add_argument("--densities", default="0.0005,0.001,0.002,0.005,0.01,0.02,0.04,0.08")
args = ap.parse_args()
m = args.m
d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
ctx = G.Context(0)
w0 = synth.gather_regime(m=m, n=1, n_test=1)
D = ctx.gram(G.BASE_GAUSSIAN, d(w0.Xd), gamma=w0.gamma)
T = ctx.gram(G.BASE_GAUSSIAN, d(w0.Xt), gamma=w0.gamma)
kron = G.gvt_kernel_terms(G.KRONECKER)
rng = np.random.default_rng(11)
for dens in (float(x) for x in args.densities.split(",")):
    n = int(dens * m * m)
    f, s = d(rng.integers(0, m, n).astype(np.int32)), d(rng.integers(0, m, n).astype(np.int32))
    a = d(synth.random_vector(1, n))
    u = torch.empty(n, dtype=torch.float32, device="cuda")
    row = {"density": dens, "n": n}
    for name, eng in (("sparse", G.ENGINE_SPARSE), ("dense", G.ENGINE_DENSE), ("auto", G.ENGINE_AUTO)):
        ctx.set_option(G.OPT_ENGINE, eng)
        ctx.matvec(D, T, f, s, f, s, a, kron, out=u)
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.matvec(D, T, f, s, f, s, a, kron, out=u)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        row[name + "_ms"] = round(float(np.median(ts)), 3)
        if name == "auto":
            row["auto_engine"] = {1: "sparse", 2: "dense"}.get(ctx.stats()["last_engine"])
    row["best"] = "sparse" if row["sparse_ms"] < row["dense_ms"] else "dense"
    print(json.dumps(row), flush=True)
    del f, s, a, u
    torch.cuda.empty_cache()
