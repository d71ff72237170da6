"""Gram GEMM throughput at C5 size: 20 000 x 20 000 Gaussian and linear Grams of dim-128 features
(CUDA events, mean of 5 after 2 warm-ups).  usage: python scripts/gram_probe.py"""
import sys, os, torch, numpy as np, json
sys.path.insert(0, os.getcwd())
import paper_2009_01054_b200 as G
ctx = G.Context(0)
X = torch.randn(20000, 128, device="cuda")
out = torch.empty(20000, 20000, device="cuda")
for kind in (G.BASE_GAUSSIAN, G.BASE_LINEAR):
    for _ in range(2): ctx.gram(kind, X, gamma=1/128, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): ctx.gram(kind, X, gamma=1/128, out=out)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"kind": kind, "ms": e0.elapsed_time(e1) / 5}))
