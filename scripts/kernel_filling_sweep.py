"""The paper's kernel-filling experiment shape on one B200 (Figure 4): for N
training pairs over a homogeneous object set (synthetic stand-in, synth.kernel_filling; Tanimoto
base kernel) and each pairwise kernel of the experiment, run the paper's protocol -- early-stopping
MINRES on 75 % inner / 25 % validation (validation AUC, patience 10), then the final fit on all
training pairs for the best iteration count -- and record iterations, GPU time and AUC.

  python scripts/kernel_filling_sweep.py [--sizes 1000,4000,...] > rows.jsonl
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

KERNELS = {"linear": G.LINEAR, "poly2d": G.POLY2D, "kronecker": G.KRONECKER, "cartesian": G.CARTESIAN,
           "symmetric": G.SYMMETRIC, "mlpk": G.MLPK}

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="1000,4000,16000,64000,256000,1024000")
ap.add_argument("--patience", type=int, default=10)
ap.add_argument("--max-iter", type=int, default=300)
args = ap.parse_args()
d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


ctx = G.Context(0)
ctx.set_option(G.OPT_SOLVER, G.SOLVER_MINRES)
for n in [int(v) for v in args.sizes.split(",")]:
    w, vlab = synth.kernel_filling(n)
    D, gram_ms = timed(lambda: ctx.gram(G.BASE_TANIMOTO, d(w.Xd)))
    f, s, y = d(w.train_first), d(w.train_second), d(w.y)
    vf, vs, vl = d(w.test_first), d(w.test_second), d(vlab)
    af, as_ = torch.cat([f, vf]), torch.cat([s, vs])
    ay = torch.cat([y, vl])
    for name, k in KERNELS.items():
        terms = G.gvt_kernel_terms(k)
        T = None if k in G.HOMOGENEOUS_KERNELS else D
        # warm (plans, workspaces), then the timed protocol
        ctx.fit_early_stopping(D, T, f, s, y, vf, vs, vl, terms, w.lam, args.patience, 3)
        (a, best, best_auc, iters, hist), es_ms = timed(
            lambda: ctx.fit_early_stopping(D, T, f, s, y, vf, vs, vl, terms, w.lam, args.patience, args.max_iter))
        ctx.fit(D, T, af, as_, ay, terms, w.lam, 3, want_history=False, raise_on_breakdown=False)  # warm
        (_, it2, _, _), fit_ms = timed(
            lambda: ctx.fit(D, T, af, as_, ay, terms, w.lam, max(best, 1), want_history=False,
                            raise_on_breakdown=False))
        row = {"n_train": int(w.n + len(vlab)), "n_inner": w.n, "n_val": len(vlab), "objects_used":
               int(np.unique(np.concatenate([w.train_first, w.train_second])).size), "kernel": name,
               "best_iter": best, "val_auc": round(best_auc, 4), "es_iters": iters, "es_ms": round(es_ms, 2),
               "es_ms_per_iter": round(es_ms / max(iters, 1), 3), "final_fit_ms": round(fit_ms, 2),
               "gram_ms": round(gram_ms, 3), "engine": {1: "sparse", 2: "dense"}.get(ctx.stats()["last_engine"], "ones-terms only")}
        print(json.dumps(row), flush=True)
