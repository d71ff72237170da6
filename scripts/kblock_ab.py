"""C4 MLPK fit time with and without the block-sparse stage 1 (GVT_OPT_KBLOCK_SKIP)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01054_b200 as G  # noqa: E402
import synth  # noqa: E402

d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
w = synth.union_domain(synth.config4())
ctx = G.Context(0)
D = ctx.gram(w.base, d(w.Xd), gamma=w.gamma)
terms = G.gvt_kernel_terms(G.MLPK)
f, s, y = d(w.train_first), d(w.train_second), d(w.y)
for rnd in range(2):
    for skip in (0, 1):
        ctx.set_option(G.OPT_KBLOCK_SKIP, skip)
        ctx.fit(D, None, f, s, y, terms, w.lam, 3, want_history=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.fit(D, None, f, s, y, terms, w.lam, w.iters, want_history=False)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"round": rnd, "kblock_skip": skip, "fit_ms": round(e0.elapsed_time(e1), 2)}), flush=True)
