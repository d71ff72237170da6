"""Gather-regime stage 2 on C5 (north star: "stage-2 gather/dot at >= 60% of B200 HBM").

Runs the C5 prediction pass (2e7 test pairs against the 1e8 training pairs, m = q = 20 000) on
the SPARSE engine, whose stage 2 is the gathered row dot u_i = <D[d_i, :], S[t_i, :]> over
S (20 000 x 20 000 fp32 = 1.6 GB, far above the 126 MB L2).  Times stage 1 / stage 2 with the
library's per-kernel CUDA events and reports the gather's achieved bandwidth against its
compulsory row bytes (8 * m_in per output: one D row + one S row of 4-byte floats; D rows are
reused across the row-sorted outputs, so the true DRAM bytes are lower -- ncu reports them).
usage: python scripts/gather_probe.py [--n-test N]   (run under ncu -k regex:k_stage2_gather)
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

ap = argparse.ArgumentParser()
ap.add_argument("--n-test", type=int, default=20_000_000)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
w = synth.config5(n_test=args.n_test)
d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
ctx = G.Context(0)
D = ctx.gram(w.base, d(w.Xd), gamma=w.gamma)
T = ctx.gram(w.base, d(w.Xt), gamma=w.gamma)
kron = G.gvt_kernel_terms(G.KRONECKER)
a = d(synth.random_vector(0, w.n))
f, s, tf, ts = d(w.train_first), d(w.train_second), d(w.test_first), d(w.test_second)
ctx.set_option(G.OPT_ENGINE, G.ENGINE_SPARSE)
out = torch.empty(w.n_test, dtype=torch.float32, device="cuda")
ctx.predict(D, T, tf, ts, f, s, a, kron, out=out)  # warm-up (plans, workspaces)
torch.cuda.synchronize()
ctx.reset_stats()
ctx.set_option(G.OPT_PROFILE, 1)
for _ in range(args.reps):
    ctx.predict(D, T, tf, ts, f, s, a, kron, out=out)
torch.cuda.synchronize()
st = ctx.stats()
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json")))
g = st["kinds"].get("stage2_gather", {"ms": float("nan"), "count": 1})
ms = g["ms"] / g["count"]
row_bytes = 8.0 * w.m * w.n_test
res = {"n_test": w.n_test, "m_in": w.m, "stage2_gather_ms": ms, "stage1_sparse_ms":
       st["kinds"].get("stage1_sparse", {"ms": float("nan")})["ms"] / args.reps,
       "compulsory_row_GB": row_bytes / 1e9, "row_bytes_GBps": row_bytes / (ms * 1e-3) / 1e9,
       "hbm_peak_GBps": peaks["hbm_gbs"], "kinds": {k: round(v["ms"] / args.reps, 3) for k, v in st["kinds"].items()}}
print(json.dumps(res))
