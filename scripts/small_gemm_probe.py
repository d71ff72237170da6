"""Fixed cost of the CTA-pair stage-1 GEMM on small complete-grid problems: per-launch stage1_tc
(library CUDA events, eager) for several (m, q).  usage: python scripts/small_gemm_probe.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01054_b200 as G  # noqa: E402

d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
ctx = G.Context(0)
ctx.set_option(G.OPT_ENGINE, G.ENGINE_DENSE)
ctx.set_option(G.OPT_STAGE2, 2)
kron = G.gvt_kernel_terms(G.KRONECKER)
rng = np.random.default_rng(0)
for m, q in ((68, 64), (68, 442), (68, 2048), (256, 442), (512, 442), (68, 4096)):
    D = ctx.gram(G.BASE_LINEAR, d(rng.standard_normal((m, 8)).astype(np.float32)))
    T = ctx.gram(G.BASE_LINEAR, d(rng.standard_normal((q, 8)).astype(np.float32)))
    f = d(np.repeat(np.arange(m, dtype=np.int32), q))
    s = d(np.tile(np.arange(q, dtype=np.int32), m))
    a = d(rng.standard_normal(m * q).astype(np.float32))
    for _ in range(3):
        ctx.matvec(D, T, f, s, f, s, a, kron)
    torch.cuda.synchronize()
    ctx.reset_stats()
    ctx.set_option(G.OPT_PROFILE, 1)
    for _ in range(20):
        ctx.matvec(D, T, f, s, f, s, a, kron)
    torch.cuda.synchronize()
    ctx.set_option(G.OPT_PROFILE, 0)
    st = ctx.stats()["kinds"]
    print(json.dumps({"m": m, "q": q, **{k: round(v["ms"] / v["count"] * 1000, 1) for k, v in st.items()}}))
