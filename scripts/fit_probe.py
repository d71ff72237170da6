"""One config's fit, for ncu launch lists and per-iteration timing (graph replay).
usage: python scripts/fit_probe.py C3 symmetric [iters] [reps]
Prints the per-iteration slope (CUDA events) between iters/2 and iters iterations."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01054_b200 as G  # noqa: E402
import synth  # noqa: E402

d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
cfg, kname = sys.argv[1], sys.argv[2]
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
w = synth.by_name(cfg)
kernel = getattr(synth, kname.upper())
if kernel in synth.HOMOGENEOUS_KERNELS and w.Xt is not None:
    w = synth.union_domain(w)
ctx = G.Context(0)
for kv in os.environ.get("GVT_PROBE_OPTS", "").split(","):
    if kv:
        k, v = kv.split("=")
        ctx.set_option(getattr(G, k), int(v))
D = ctx.gram(w.base, d(w.Xd), gamma=w.gamma, coef0=w.coef0, degree=w.degree)
T = None if w.Xt is None else ctx.gram(w.base, d(w.Xt), gamma=w.gamma, coef0=w.coef0, degree=w.degree)
terms = G.gvt_kernel_terms(kernel)
f, s, y = d(w.train_first), d(w.train_second), d(w.y)
ts = {}
for k in (iters // 2, iters):
    best = 1e30
    for _ in range(reps):
        ctx.fit(D, T, f, s, y, terms, w.lam, k, want_history=False, raise_on_breakdown=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.fit(D, T, f, s, y, terms, w.lam, k, want_history=False, raise_on_breakdown=False)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    ts[k] = best
print(json.dumps({"config": cfg, "kernel": kname, "engine": ctx.stats()["last_engine"],
                  "us_per_iter": round(1e3 * (ts[iters] - ts[iters // 2]) / (iters - iters // 2), 2),
                  "fit_ms": {str(k): round(v, 3) for k, v in ts.items()}}), flush=True)
