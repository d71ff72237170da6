"""Phase timing of the persistent small solver on C2 for each barrier mode (GVT_SMALL_BAR: bit 0 =
two-level arrival, bit 1 = sleep while polling), one process per mode, with GVT_SMALL_PROF phase stamps.
usage: python scripts/small_bar_probe.py"""
import os
import subprocess
import sys

CHILD = r"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import synth, paper_2009_01054_b200 as G
w = synth.config2(); ctx = G.Context(0)
d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
D = ctx.gram(w.base, d(w.Xd), gamma=w.gamma); T = ctx.gram(w.base, d(w.Xt), gamma=w.gamma)
f, s, y = d(w.train_first), d(w.train_second), d(w.y); kron = G.gvt_kernel_terms(G.KRONECKER)
ctx.set_option(G.OPT_ENGINE, 4)
def t(k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record(); ctx.fit(D, T, f, s, y, kron, w.lam, k, want_history=False); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
t(10)
print("us_per_iter", round(1e3 * (t(100) - t(10)) / 90, 2), flush=True)
"""
for mode in (0, 1, 2, 3):
    env = dict(os.environ, GVT_SMALL_BAR=str(mode))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(f"mode {mode}: {r.stdout.strip()}", flush=True)
    env["GVT_SMALL_PROF"] = "1"
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print("\n".join(r.stderr.strip().splitlines()[-2:]), flush=True)
