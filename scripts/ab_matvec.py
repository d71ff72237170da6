"""A/B timing of the C5 fit loop between configurations on the same box.

  python scripts/ab_matvec.py "cta=1" "cta=2" [--rounds 2]      # option sets (GVT options)
  python scripts/ab_matvec.py "lib=ab/libA.so" "lib=ab/libB.so"  # library builds
  python scripts/ab_matvec.py "gm=16" "gm=8" "gm=4"              # GEMM rasterization group (GVT_GROUP_M)
  python scripts/ab_matvec.py "E_GVT_BUILD_CHUNKS=0" "E_GVT_BUILD_CHUNKS=1"  # any library environment knob

Each round runs one subprocess per configuration that times a 10-iteration fit at C5
(CUDA events) after warm-up, reporting ms and per-kernel ms/launch with the SM clock
sampled by nvidia-smi, so A and B see the same thermal/power state.
"""
import os
import subprocess
import sys

CHILD = r"""
import json, os, sys, subprocess, numpy as np, torch
sys.path.insert(0, os.getcwd())
import synth, paper_2009_01054_b200 as G
spec = dict(kv.split("=") for kv in sys.argv[1].split(",") if kv)
w = synth.config5()
ctx = G.Context(0)
if "cta" in spec: ctx.set_option(G.OPT_GEMM_CTA, int(spec["cta"]))
if "prec" in spec: ctx.set_option(G.OPT_TC_PRECISION, int(spec["prec"]))
if "sf" in spec: ctx.set_option(G.OPT_SORTED_FIT, int(spec["sf"]))
d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
D = ctx.gram(w.base, d(w.Xd), gamma=w.gamma); T = ctx.gram(w.base, d(w.Xt), gamma=w.gamma)
f, s = d(w.train_first), d(w.train_second); a = d(synth.random_vector(0, w.n)); u = torch.empty_like(a)
kron = G.gvt_kernel_terms(G.KRONECKER)
for _ in range(2): ctx.fit(D, T, f, s, a, kron, 1.0, 3, out=u, want_history=False, raise_on_breakdown=False)
torch.cuda.synchronize(); ctx.reset_stats(); ctx.set_option(G.OPT_PROFILE, 1)
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "200"],
                       stdout=subprocess.PIPE, text=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); ctx.fit(D, T, f, s, a, kron, 1.0, 10, out=u, want_history=False, raise_on_breakdown=False); e1.record(); torch.cuda.synchronize()
smi.terminate(); rows = [l.split(",") for l in smi.stdout.read().strip().splitlines()]
clk = [float(r[0]) for r in rows if len(r) > 1]; pw = [float(r[1]) for r in rows if len(r) > 1]
st = ctx.stats()
print(json.dumps({"fit10_ms": round(e0.elapsed_time(e1), 1), "sm_mhz": float(np.median(clk)) if clk else None,
                  "power_w": float(np.median(pw)) if pw else None,
                  "kinds": {k: round(v["ms"] / max(1, v["count"]), 3) for k, v in st["kinds"].items()
                            if k.startswith("stage") or k in ("densify", "plan_sort(cub)", "plan_gather")}}))
"""


def main():
    specs = [a for a in sys.argv[1:] if not a.startswith("--")]
    rounds = 2
    if "--rounds" in sys.argv:
        rounds = int(sys.argv[sys.argv.index("--rounds") + 1])
        specs = [s for s in specs if s != str(rounds)]
    for r in range(rounds):
        for spec in specs:
            env = dict(os.environ)
            kv = dict(x.split("=") for x in spec.split(",") if x)
            if "lib" in kv:
                env["GVT_LIBRARY"] = os.path.abspath(kv["lib"])
            if "gm" in kv:  # rasterization group of the CTA-pair GEMM
                env["GVT_GROUP_M"] = kv["gm"]
            if "rs" in kv:  # fp16 S with per-row bound scales (1) or per-(row, 256-col tile) scales (0)
                env["GVT_S16_ROWSCALE"] = kv["rs"]
            for k, v in kv.items():  # E_NAME=V: any environment knob of the library (e.g. E_GVT_BUILD_CHUNKS=0)
                if k.startswith("E_"):
                    env[k[2:]] = v
            if "l2" in kv:  # TMA L2 promotion of the GEMM operand maps (0 none, 1 64B, 2 128B, 3 256B)
                env["GVT_L2PROMO"] = kv["l2"]
            out = subprocess.run([sys.executable, "-c", CHILD, spec], env=env, capture_output=True, text=True)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-1500:]
            print(f"round {r} [{spec}]: {line}", flush=True)


if __name__ == "__main__":
    main()
