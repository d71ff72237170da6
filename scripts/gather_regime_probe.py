"""Gather regime at C5 scale (north star: "stage-2 gather/dot at >= 60% of B200 HBM bandwidth").

SURVEY 8(d): below ~2-3 % pair density (Heterodimer-like, 0.2 %) the GVT stage 2 is the row
gather u_i = <A[r_i, :], S[c_i, :]>, HBM-bound at 8 * m_in bytes per output.  This probe
instantiates that regime at the C5 object counts so that S (q x m_in fp32 = 1.6 GB) and the Gram
factors (1.6 GB each) are far above the 126 MB L2:

  m = q = 20 000 objects, dim 128 N(0,1) features, Gaussian gamma = 1/128 (S5);
  n_train uniform pairs (default 8e5 = 0.2 % of the grid), n_test uniform test pairs (2e6);
  a ~ N(0, 1).  Seeded (synth.gather_regime, PCG64 seed 7).

The auto engine picks the sparse path at this density (by its time estimate).  Times, with the
library's per-kernel CUDA events: the training matvec (stage 1 + gather over n_train outputs) and
the prediction (stage 1 + gather over n_test outputs).  Reports the gather's achieved bandwidth
against its algorithmic bytes (8 * m_in per output: one A row + one S row, fp32) and the measured
HBM peak.  usage: python scripts/gather_regime_probe.py [--n-train N] [--n-test N] [--reps R]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_01054_b200 as G  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=20_000)
ap.add_argument("--n-train", type=int, default=800_000)
ap.add_argument("--n-test", type=int, default=2_000_000)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--engine", type=int, default=0, help="GVT_OPT_ENGINE (0 auto, 1 sparse, 2 dense)")
args = ap.parse_args()

w = synth.gather_regime(m=args.m, n=args.n_train, n_test=args.n_test)
m = q = args.m
Xd, Xt, f, s, tf, ts = w.Xd, w.Xt, w.train_first, w.train_second, w.test_first, w.test_second
a_h = synth.random_vector(0, args.n_train)

d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
ctx = G.Context(0)
ctx.set_option(G.OPT_ENGINE, args.engine)
D = ctx.gram(G.BASE_GAUSSIAN, d(Xd), gamma=1.0 / 128)
T = ctx.gram(G.BASE_GAUSSIAN, d(Xt), gamma=1.0 / 128)
kron = G.gvt_kernel_terms(G.KRONECKER)
f, s, tf, ts, a = d(f), d(s), d(tf), d(ts), d(a_h)
u = torch.empty(args.n_train, dtype=torch.float32, device="cuda")
out = torch.empty(args.n_test, dtype=torch.float32, device="cuda")
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
res = {"m": m, "q": q, "n_train": args.n_train, "n_test": args.n_test,
       "density": args.n_train / (m * q), "hbm_peak_GBps": peaks["hbm_gbs"]}
for name, call, n_out in (("matvec", lambda: ctx.matvec(D, T, f, s, f, s, a, kron, out=u), args.n_train),
                          ("predict", lambda: ctx.predict(D, T, tf, ts, f, s, a, kron, out=out), args.n_test)):
    call()  # warm-up: plans, workspaces
    torch.cuda.synchronize()
    ctx.reset_stats()
    ctx.set_option(G.OPT_PROFILE, 1)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.reps):
        call()
    ev1.record()
    torch.cuda.synchronize()
    ctx.set_option(G.OPT_PROFILE, 0)
    st = ctx.stats()
    kinds = {k: round(v["ms"] / args.reps, 3) for k, v in st["kinds"].items()}
    g = st["kinds"].get("stage2_gather")
    r = {"ms": ev0.elapsed_time(ev1) / args.reps, "engine": st.get("last_engine"), "kinds": kinds}
    if g:
        gms = g["ms"] / g["count"]
        alg = 8.0 * m * n_out
        r.update({"gather_ms": gms, "gather_alg_GB": alg / 1e9, "gather_GBps": alg / (gms * 1e-3) / 1e9,
                  "gather_frac_hbm": alg / (gms * 1e-3) / 1e9 / peaks["hbm_gbs"]})
    r["Gpairs_per_s"] = n_out / (r["ms"] * 1e-3) / 1e9
    res[name] = r
print(json.dumps(res))
