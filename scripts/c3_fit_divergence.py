"""Diagnosis: C3 Symmetric fit weights with the round-2 fast paths (split-K, warp-per-row X build) vs without,
after 2/5/10/20 CG iterations (fp32 rounding-order differences amplified by the Krylov recurrence)."""
import sys, os, numpy as np, subprocess, json, tempfile
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import importlib.util
spec = importlib.util.spec_from_file_location("t", "tests/test_gpu_round2_paths.py")
t = importlib.util.module_from_spec(spec); spec.loader.exec_module(t)
import pathlib
tmp = pathlib.Path(tempfile.mkdtemp())
for it in (2, 5, 10, 20):
    a, ea = t.run("C3", "symmetric", "fit", it, {}, tmp, "a")
    b, eb = t.run("C3", "symmetric", "fit", it, {"GVT_SPLITK": "0", "GVT_BUILD_WARP": "0"}, tmp, "b")
    c, ec = t.run("C3", "symmetric", "fit", it, {"GVT_SPLITK": "0"}, tmp, "c")
    print(it, "rel(split+warp, plain)=%.2e rel(warp, plain)=%.2e" % (t.rel(a, b), t.rel(c, b)), ea["relres"], eb["relres"], ec["relres"], flush=True)
