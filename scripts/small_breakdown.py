"""Per-kernel breakdown of one solver iteration on the small configs (eager launches with the
library's per-kernel CUDA events, GVT_OPT_PROFILE = 1), next to the graph-replayed marginal cost.
usage: python scripts/small_breakdown.py [C2:kronecker C3:symmetric C4:ranking ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01054_b200 as G  # noqa: E402
import synth  # noqa: E402

d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
specs = sys.argv[1:] or ["C1:kronecker", "C2:kronecker", "C3:symmetric", "C3:cartesian", "C4:poly2d", "C4:ranking"]
for spec in specs:
    cfg, kname = spec.split(":")
    w = synth.by_name(cfg)
    kernel = getattr(synth, kname.upper())
    if kernel in synth.HOMOGENEOUS_KERNELS and w.Xt is not None:
        w = synth.union_domain(w)
    terms = G.gvt_kernel_terms(kernel)
    ctx = G.Context(0)
    D = ctx.gram(w.base, d(w.Xd), gamma=w.gamma)
    T = None if w.Xt is None else ctx.gram(w.base, d(w.Xt), gamma=w.gamma)
    f, s, y = d(w.train_first), d(w.train_second), d(w.y)
    K = 20
    ctx.fit(D, T, f, s, y, terms, w.lam, K, want_history=False)
    torch.cuda.synchronize()
    # graph-replayed marginal cost
    ts = {}
    for k in (10, 30):
        ctx.fit(D, T, f, s, y, terms, w.lam, k, want_history=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.fit(D, T, f, s, y, terms, w.lam, k, want_history=False)
        e1.record()
        torch.cuda.synchronize()
        ts[k] = e0.elapsed_time(e1)
    marg = 1e3 * (ts[30] - ts[10]) / 20
    # eager, per-kernel events: difference of a 30- and a 10-iteration fit = 20 iterations
    kinds = {}
    for k, sign in ((30, 1), (10, -1)):
        ctx.reset_stats()
        ctx.set_option(G.OPT_PROFILE, 1)
        ctx.fit(D, T, f, s, y, terms, w.lam, k, want_history=False)
        torch.cuda.synchronize()
        st = ctx.stats()
        ctx.set_option(G.OPT_PROFILE, 0)
        for name, v in st["kinds"].items():
            e = kinds.setdefault(name, [0.0, 0])
            e[0] += sign * v["ms"]
            e[1] += sign * v["count"]
    per_iter = {k: {"us": round(1e3 * v[0] / 20, 2), "launches": v[1] / 20} for k, v in kinds.items() if v[1] > 0}
    print(json.dumps({"config": cfg, "kernel": kname, "engine": st["last_engine"], "graph_marginal_us": round(marg, 2),
                      "eager_per_iter": per_iter,
                      "eager_sum_us": round(sum(v["us"] for v in per_iter.values()), 2)}), flush=True)
    ctx.close()
