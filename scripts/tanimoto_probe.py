"""Tanimoto Gram throughput: m x m for 0/1 fingerprints of `dim` bits (POPC/AND word ops)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01054_b200 as G  # noqa: E402

ctx = G.Context(0)
rng = np.random.default_rng(0)
for m, dim in [(2967, 1024), (20000, 2048)]:
    X = torch.from_numpy((rng.uniform(size=(m, dim)) < 0.1).astype(np.float32)).cuda()
    K = ctx.gram(G.BASE_TANIMOTO, X)
    ctx.reset_stats()
    ctx.set_option(G.OPT_PROFILE, 1)
    for _ in range(3):
        ctx.gram(G.BASE_TANIMOTO, X, out=K)
    torch.cuda.synchronize()
    st = ctx.stats()
    ctx.set_option(G.OPT_PROFILE, 0)
    ms = st["kinds"]["gram_simt"]["ms"] / 3
    words = m * m * ((dim + 31) // 32)
    print(json.dumps({"m": m, "dim": dim, "ms": round(ms, 3), "Gword_ops_per_s": round(words / ms / 1e6, 1)}))
