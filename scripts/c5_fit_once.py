"""One short C5 fit (3 iterations) on the library in-tree: a target for ncu kernel captures.
usage: ncu -k regex:<kernel> -c 1 python scripts/c5_fit_once.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01054_b200 as G  # noqa: E402
import synth  # noqa: E402

w = synth.config5()
ctx = G.Context(0)
d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
D = ctx.gram(w.base, d(w.Xd), gamma=w.gamma)
T = ctx.gram(w.base, d(w.Xt), gamma=w.gamma)
f, s, y = d(w.train_first), d(w.train_second), d(w.y)
a = torch.empty_like(y)
ctx.fit(D, T, f, s, y, G.gvt_kernel_terms(G.KRONECKER), w.lam, 3, out=a, want_history=False)
torch.cuda.synchronize()
print("ok")
