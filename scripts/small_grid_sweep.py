"""C2 fit time per iteration on the persistent small solver (engine 4) against its CTA count
(GVT_SMALL_GRID, one process per setting) next to the multi-kernel dense engine.
usage: python scripts/small_grid_sweep.py"""
import json
import os
import subprocess
import sys

CHILD = r"""
import json, os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import synth, paper_2009_01054_b200 as G
w = synth.config2(); ctx = G.Context(0)
d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
D = ctx.gram(w.base, d(w.Xd), gamma=w.gamma); T = ctx.gram(w.base, d(w.Xt), gamma=w.gamma)
f, s, y = d(w.train_first), d(w.train_second), d(w.y); kron = G.gvt_kernel_terms(G.KRONECKER)
ctx.set_option(G.OPT_ENGINE, int(sys.argv[1]))
def t(k):
    ctx.fit(D, T, f, s, y, kron, w.lam, k, want_history=False); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record(); ctx.fit(D, T, f, s, y, kron, w.lam, k, want_history=False); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
t10, t100 = t(10), t(100)
print(json.dumps({"engine": int(sys.argv[1]), "grid": os.environ.get("GVT_SMALL_GRID"), "fit100_ms": round(t100, 3),
                  "us_per_iter": round(1e3 * (t100 - t10) / 90, 2), "last_engine": ctx.stats()["last_engine"]}))
"""
for engine, grids in ((2, [None]), (4, [None, 16, 32, 64, 96, 128])):
    for g in grids:
        env = dict(os.environ)
        if g:
            env["GVT_SMALL_GRID"] = str(g)
        r = subprocess.run([sys.executable, "-c", CHILD, str(engine)], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-800:], flush=True)
