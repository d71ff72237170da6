"""C5 fit of a few iterations (for ncu captures of the dense GEMMs in their fit configuration)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01054_b200 as G  # noqa: E402
import synth  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = synth.config5()
d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
ctx = G.Context(0)
ctx.set_option(G.OPT_GRAPHS, 0)
D = ctx.gram(w.base, d(w.Xd), gamma=w.gamma)
T = ctx.gram(w.base, d(w.Xt), gamma=w.gamma)
kron = G.gvt_kernel_terms(G.KRONECKER)
a, it, _, _ = ctx.fit(D, T, d(w.train_first), d(w.train_second), d(w.y), kron, w.lam, iters, want_history=False)
torch.cuda.synchronize()
print("fit iters", it)
