"""Per-iteration solver cost on a config (graph replay): the slope of fit time over the iteration
count, for each solver form.  usage: python scripts/iter_cost.py C1 [C2 ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01054_b200 as G  # noqa: E402
import synth  # noqa: E402

d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
for name in sys.argv[1:]:
    w = synth.by_name(name)
    ctx = G.Context(0)
    D = ctx.gram(w.base, d(w.Xd), gamma=w.gamma)
    T = None if w.Xt is None else ctx.gram(w.base, d(w.Xt), gamma=w.gamma)
    terms = G.gvt_kernel_terms(w.kernels[0])
    f, s, y = d(w.train_first), d(w.train_second), d(w.y)
    out = {}
    for label, solver, variant in (("cg-hs", 0, 0), ("cg-cgg", 0, 1), ("minres", 1, 0)):
        ctx.set_option(G.OPT_SOLVER, solver)
        ctx.set_option(G.OPT_CG_VARIANT, variant)
        ts = {}
        for k in (10, 90):
            ctx.fit(D, T, f, s, y, terms, w.lam, k, want_history=False, raise_on_breakdown=False)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.fit(D, T, f, s, y, terms, w.lam, k, want_history=False, raise_on_breakdown=False)
            e1.record()
            torch.cuda.synchronize()
            ts[k] = e0.elapsed_time(e1)
        out[label] = {"us_per_iter": round(1e3 * (ts[90] - ts[10]) / 80, 2), "fixed_ms": round(ts[10], 3)}
    print(json.dumps({"config": name, **out}), flush=True)
    ctx.close()
