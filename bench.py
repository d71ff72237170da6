"""bench.py -- GVT hot-path benchmark (BASELINE.json metric: "GVT matvec Gpairs/s and CG
iters/s at 1/2/4/8 B200; % of HBM roofline").

One STEP = one pass of the whole hot path over the workload:
base-kernel Grams D, T from the object features (a2), pairwise_krr_fit = plan + `iters` CG
iterations of the GVT matvec (a1, a3-a9), pairwise_predict over the test pairs (a10).
value = matvec pair-rows delivered per second over the whole step,
        (iters * n_train + n_test) / t_step, in Gpairs/s (whole job, all ranks).

Default workload: C5 (BASELINE.json configs[4], the metric's 1/2/4/8-GPU config; it fits
one B200).  Inputs (1e8 pairs = 0.8 GB of ids) exceed the 126 MB L2, so no flush is
needed between steps.  --impl reference times the fp64 oracle (oracle/, test
infrastructure) on a bounded sample of the same workload on the host cores.

Launch: python bench.py [--gpus N --steps K --warmup W]; for N > 1 under
torch.distributed.run (one rank per GPU, NCCL); rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "GVT matvec Gpairs/s and CG iters/s at 1/2/4/8 B200; % of HBM roofline"
UNIT = "Gpairs/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "bf16_tflops": d.get("bf16_tflops", 1590.0),
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", 1400.0),
                "sm_max_mhz": d.get("sm_max_mhz", 1965.0), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0,
            "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- workloads
def workload(name: str):
    if name == "C5":
        return synth.config5()
    if name == "C4":
        return synth.config4()
    if name == "C3":
        return synth.config3()
    if name == "C2":
        return synth.config2()
    if name == "C1":
        return synth.config1()
    if name.startswith("C5s"):       # scaled-down C5 for quick runs: C5s<n_millions>
        n = int(float(name[3:]) * 1e6)
        return synth.config5(n=n, n_test=max(1, n // 5), m=max(200, int(20000 * (n / 1e8) ** 0.5)))
    raise ValueError(name)


def default_kernel(w):
    return w.kernels[0]


def config_dict(args, w, kernel, world):
    """The workload's `config` object, identical in both arms (the GPU arm and --impl reference)."""
    return {"workload": args.workload, "kernel": synth.KERNEL_NAMES[kernel], "n_train": w.n, "n_test": w.n_test,
            "m": w.m, "q": w.q, "cg_iters": w.iters, "lambda": w.lam,
            "engine": {0: "auto", 1: "sparse", 2: "dense"}[args.engine], "tc_precision": args.precision,
            "exchange": ["S-allgather", "u-reduce", "auto (by estimated bytes)"][args.exchange],
            "comm": args.comm if world > 1 else None, "solver": args.solver,
            "cg_variant": ["hestenes-stiefel", "chronopoulos-gear"][args.cg_variant],
            "l2": "inputs (pair ids 0.8 GB at C5) larger than the 126 MB L2; no flush",
            "step": "gram(D)+gram(T)+pairwise_krr_fit(iters)+pairwise_predict"}


# ----------------------------------------------------------------------------- roofline
def _traffic(kernel_kind):
    """DRAM bytes per launch of `kernel_kind` from the committed ncu --set full capture
    (profiles/r02_traffic.json), or None."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_traffic.json")) as fh:
            rec = json.load(fh).get(kernel_kind)
        return int(rec["bytes"]) if rec else None
    except (OSError, ValueError, KeyError):
        return None


def roofline(kinds: dict, w, kernel, launches_per_step: dict, peaks: dict, engine: int, precision: str = "fp16x3"):
    """Dominant kernel (largest summed event time) vs its roof.  Algorithmic work per
    launch: stage 1 = q_out FMA per pair-matrix entry, stage 2 = m_in FMA
    per output; dense engine reports against the TF32 tensor peak (measured bf16 x 0.5),
    sparse/SIMT kernels against the fp32 ALU peak (148 SM x 128 lanes x 2 x f_max)."""
    if not kinds:
        return None
    name, rec = max(kinds.items(), key=lambda kv: kv[1]["ms"])
    per_launch_ms = rec["ms"] / max(1, rec["count"])
    n, n_test, m, q = w.n, w.n_test, w.m, w.q
    nnz = n * {synth.SYMMETRIC: 2, synth.ANTISYMMETRIC: 2, synth.MLPK: 4}.get(kernel, 1)
    alu_peak = 148 * 128 * 2 * peaks["sm_max_mhz"] * 1e6 / 1e12  # TFLOP/s
    cnt = rec["count"]
    fit_launches = max(1, w.iters)
    if name in ("stage1_sparse", "stage1_tc"):
        # (iters fit launches over n pairs) + (1 predict launch over n pairs): same per-launch work
        flops = 2.0 * q * nnz
    elif name in ("stage2_gather", "stage2_tc"):
        # fit launches: n outputs; predict: n_test outputs -> average per launch
        fl_fit = 2.0 * m * n
        fl_pred = 2.0 * m * n_test
        steps = cnt / (fit_launches + 1)
        flops = (fl_fit * fit_launches + fl_pred) * steps / cnt
    else:
        return {"kernel": name, "bound": None, "achieved": None, "peak": None, "unit": None, "frac": None,
                "traffic": None}
    achieved = flops / (per_launch_ms * 1e-3) / 1e12
    out = {"kernel": name, "ms_per_launch": round(per_launch_ms, 4), "launches": cnt}
    traffic = _traffic(name)
    if name.endswith("_tc"):
        # the dense engine runs 3 tensor-core products over the dense M x N x K GEMM
        M, N, K = (q, m, q) if name.startswith("stage1") else (m, q, m)
        executed = 3 * 2.0 * M * N * K / (per_launch_ms * 1e-3) / 1e12
        if precision == "fp16x3":
            peak, src = peaks["bf16_tflops_sustained"], f"fp16/bf16 dense, measured sustained ({peaks['source']})"
        else:
            peak, src = peaks["bf16_tflops_sustained"] * 0.5, f"tf32 = 0.5 x measured bf16 sustained ({peaks['source']})"
        out.update({"bound": "tensor", "achieved": round(achieved, 3), "peak": round(peak, 1), "unit": "TFLOP/s",
                    "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": src,
                    "achieved_basis": "algorithmic FMAs of SURVEY 8(d) (q_out per pair-matrix entry / m_in per output)",
                    "executed_tflops": round(executed, 1), "executed_frac": round(executed / peak, 4),
                    "alu_roof_frac": round(achieved / alu_peak, 4)})
        # the engine's own ceiling: a dense tile engine executes M N K products for the
        # algorithmic (density x M N K) ones, three times (3xFP16 / 3xTF32 splits), so at 100 % of the
        # tensor peak its algorithmic fraction is density / 3; fp32-accurate peak = peak / 3
        ceiling = (flops / (2.0 * M * N * K)) / 3.0
        out.update({"passes": 3, "density": round(3.0 * ceiling, 4), "ceiling_frac": round(ceiling, 4),
                    "frac_of_ceiling": round(achieved / peak / ceiling, 4),
                    "fp32_accurate_peak": round(peak / 3.0, 1),
                    "fp32_accurate_frac": round(achieved / (peak / 3.0), 4),
                    "ceiling_note": "frac = algorithmic flops / measured bf16 sustained peak; a dense 3-pass "
                                    "engine at density d cannot exceed d / 3 (ceiling_frac)"})
    else:
        out.update({"bound": "alu", "achieved": round(achieved, 3), "peak": round(alu_peak, 1), "unit": "TFLOP/s",
                    "frac": round(achieved / alu_peak, 4), "traffic": traffic,
                    "peak_source": "fp32 SIMT: 148 SM x 128 lanes x 2 x sm_max_mhz"})
    if traffic is not None:
        out["traffic_unit"] = "bytes per launch (ncu dram read + write, profiles/r02_traffic.json)"
    return out


# ----------------------------------------------------------------------------- oracle (CPU) legs
_ORACLE_GRAMS = {}


def oracle_grams(w):
    """fp64 oracle Grams of the workload, computed once per process (not part of the sample)."""
    import oracle as O
    key = w.name
    if key not in _ORACLE_GRAMS:
        D = O.gram(w.base, w.Xd, gamma=w.gamma, coef0=w.coef0, degree=w.degree)
        T = None if w.Xt is None else O.gram(w.base, w.Xt, gamma=w.gamma, coef0=w.coef0, degree=w.degree)
        _ORACLE_GRAMS[key] = (D, T)
    return _ORACLE_GRAMS[key]


def oracle_sample(w, kernel, n_targets=8, seed=0, min_seconds=1.0):
    """The oracle's GVT matvec on a bounded sample of the training matvec: the outputs whose
    second element lies among `n_targets` seeded targets (the oracle then forms S only for
    those rows: the same fraction of stage 1 and stage 2 work as of the full matvec)."""
    import oracle as O
    rng = np.random.default_rng(seed)
    tset = rng.choice(w.q, min(n_targets, w.q), replace=False)
    idx = np.nonzero(np.isin(w.train_second, tset))[0]
    D, T = oracle_grams(w)
    a = synth.random_vector(seed, w.n)
    terms = O.kernel_terms(kernel)
    # small workloads: repeat the sample until it has run for >= 1 s (outputs counted per repeat)
    reps, t0 = 0, time.perf_counter()
    while True:
        O.gvt_matvec(terms, D, T, w.train_first[idx], w.train_second[idx], w.train_first, w.train_second, a)
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= min_seconds:
            break
    return len(idx) * reps, dt, O.num_threads()


def run_reference(args, rank, world):
    if rank != 0:
        return
    w = workload(args.workload)
    kernel = default_kernel(w)
    times, cnt = [], 0
    nt = args.ref_targets
    for i in range(args.warmup + args.steps):
        k, dt, cores = oracle_sample(w, kernel, n_targets=nt, seed=i)
        if i >= args.warmup:
            times.append(dt)
            cnt += k
    tot = sum(times)
    val = cnt / tot / 1e9
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_dict(args, w, kernel, world),
            "reference_step": "a bounded sample of the training matvec (the oracle's per-term GVT, fp64) on the host "
                              "cores; the GPU arm's step is gram(D)+gram(T)+pairwise_krr_fit(iters)+pairwise_predict",
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"fp64 oracle per-term GVT training matvec restricted to the outputs of {nt} "
                                       f"seeded targets per step, repeated for >= 1 s ({cnt // max(1, args.steps)} "
                                       f"outputs per step, stage 1 over all {w.n} pairs for those rows)"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def gather_regime_leg(local_rank, peaks, reps=5):
    """North-star gather target on its own regime: the sparse
    engine at C5 object counts and 0.2 % density (synth.gather_regime), where stage 2 is the row
    gather.  Device-timed with the library's per-kernel CUDA events.  Compulsory DRAM bytes of
    the gather: one S row per output (4 * m_in B; S is 13x the L2) plus each A row once (the
    outputs are sorted by row)."""
    import torch

    import paper_2009_01054_b200 as G
    w = synth.gather_regime()
    dev = torch.device("cuda", local_rank)

    def d(x):
        return torch.from_numpy(np.ascontiguousarray(x)).to(dev)

    res = {"workload": f"gather regime: m=q={w.m}, {w.n} uniform train pairs ({w.n / (w.m * w.q):.1%} density), "
                       f"{w.n_test} uniform test pairs, Gaussian dim {w.Xd.shape[1]}, Kronecker",
           "ncu_dram": "profiles/r01_gather_regime_ncu.txt"}
    with G.Context(local_rank) as ctx:
        D = ctx.gram(w.base, d(w.Xd), gamma=w.gamma)
        T = ctx.gram(w.base, d(w.Xt), gamma=w.gamma)
        terms = G.gvt_kernel_terms(G.KRONECKER)
        f, s, tf, ts = d(w.train_first), d(w.train_second), d(w.test_first), d(w.test_second)
        a = d(synth.random_vector(0, w.n))
        u = torch.empty(w.n, dtype=torch.float32, device=dev)
        sc = torch.empty(w.n_test, dtype=torch.float32, device=dev)
        for name, call, n_out in (("matvec", lambda: ctx.matvec(D, T, f, s, f, s, a, terms, out=u), w.n),
                                  ("predict", lambda: ctx.predict(D, T, tf, ts, f, s, a, terms, out=sc), w.n_test)):
            for _ in range(3):
                call()
            torch.cuda.synchronize(dev)
            ctx.reset_stats()
            ctx.set_option(G.OPT_PROFILE, 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                call()
            e1.record()
            torch.cuda.synchronize(dev)
            ctx.set_option(G.OPT_PROFILE, 0)
            st = ctx.stats()
            g = st["kinds"]["stage2_gather"]
            gms = g["ms"] / g["count"]
            comp = 4.0 * w.m * n_out + 4.0 * w.m * w.m
            res[name] = {"ms": e0.elapsed_time(e1) / reps, "Gpairs_per_s": n_out / (e0.elapsed_time(e1) / reps * 1e-3) / 1e9,
                         "engine": {1: "sparse", 2: "dense"}.get(st["last_engine"]),
                         "stage1_sparse_ms": st["kinds"]["stage1_sparse"]["ms"] / reps, "stage2_gather_ms": gms,
                         "gather_compulsory_GB": comp / 1e9, "gather_GBps": comp / (gms * 1e-3) / 1e9,
                         "gather_frac_hbm": comp / (gms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                         "gather_row_bytes_GBps": 8.0 * w.m * n_out / (gms * 1e-3) / 1e9}
    res["hbm_peak_GBps"] = peaks["hbm_gbs"]
    return res


# per-config legs of the default line (make the C1-C4 numbers driver-observed)
CONFIG_RUNS = [("C1", "kronecker"), ("C2", "kronecker"), ("C3", "symmetric"), ("C3", "antisymmetric"),
               ("C3", "cartesian"), ("C4", "poly2d"), ("C4", "mlpk"), ("C4", "ranking")]
# SURVEY.md 8(d) floors per training matvec on one B200, T_roof = max(FMA / 37.2e12, bytes / 6.54e12);
# C1 and C2 are latency-bound (no roofline floor: "report us per iteration")
FLOORS_US = {("C3", "symmetric"): 32.0, ("C3", "antisymmetric"): 32.0, ("C3", "cartesian"): 50.0,
             ("C4", "poly2d"): 430.0, ("C4", "mlpk"): 1300.0, ("C4", "ranking"): 45.0}


def configs_leg(local_rank, steps=5, warmup=3):
    """C1-C4 (every kernel each config runs) on one GPU: the same step as the headline
    (Grams + pairwise_krr_fit(iters) + pairwise_predict, graph-replayed solver), device-timed; plus the
    solver's marginal cost per iteration (slope of the fit time between iters/2 and iters iterations)
    against the SURVEY floor of one training matvec.  Then the oracle's 1-core legs (C1-C3 training
    matvec, the per-term GVT) and the explicit-K C1 matvec, the paper's baseline."""
    import torch

    import oracle as O
    import paper_2009_01054_b200 as G
    dev = torch.device("cuda", local_rank)

    def d(x):
        return torch.from_numpy(np.ascontiguousarray(x)).to(dev)

    def timed(fn, reps=1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / reps

    cache, runs = {}, []
    for cfg, kname in CONFIG_RUNS:
        if cfg not in cache:
            cache.clear()
            cache[cfg] = synth.by_name(cfg)
        w = cache[cfg]
        kernel = getattr(synth, kname.upper())
        if kernel in synth.HOMOGENEOUS_KERNELS and w.Xt is not None:
            w = synth.union_domain(w)
        terms = G.gvt_kernel_terms(kernel)
        with G.Context(local_rank) as ctx:
            Xd, Xt = d(w.Xd), (None if w.Xt is None else d(w.Xt))
            D = torch.empty((w.m, w.m), dtype=torch.float32, device=dev)
            T = None if Xt is None else torch.empty((w.q, w.q), dtype=torch.float32, device=dev)
            f, s_, y, tf, ts = d(w.train_first), d(w.train_second), d(w.y), d(w.test_first), d(w.test_second)
            a = torch.empty(w.n, dtype=torch.float32, device=dev)
            sc = torch.empty(w.n_test, dtype=torch.float32, device=dev)

            def step(k=w.iters):
                ctx.gram(w.base, Xd, gamma=w.gamma, coef0=w.coef0, degree=w.degree, out=D)
                if T is not None:
                    ctx.gram(w.base, Xt, gamma=w.gamma, coef0=w.coef0, degree=w.degree, out=T)
                ctx.fit(D, T, f, s_, y, terms, w.lam, k, 0.0, out=a, want_history=False)
                ctx.predict(D, T, tf, ts, f, s_, a, terms, out=sc)

            for _ in range(warmup):
                step()
            torch.cuda.synchronize(dev)
            ctx.reset_stats()
            ms = timed(step, steps)
            launches = ctx.stats()["launches"] / steps
            k1, k0 = w.iters, w.iters // 2
            fit = lambda k: ctx.fit(D, T, f, s_, y, terms, w.lam, k, 0.0, out=a, want_history=False)  # noqa: E731
            fit(k0), fit(k1)
            # the engine of the fit (the step's last call is the predict, which may take another engine)
            engine = {1: "sparse", 2: "dense", 3: "single-CTA", 4: "persistent"}.get(ctx.stats()["last_engine"])
            t0 = min(timed(lambda: fit(k0)) for _ in range(3))
            t1 = min(timed(lambda: fit(k1)) for _ in range(3))
            us_iter = 1e3 * (t1 - t0) / (k1 - k0)
            floor = FLOORS_US.get((cfg, kname))
            runs.append({"config": cfg, "kernel": kname, "ms_per_step": round(ms, 4), "iters": w.iters,
                         "us_per_iter_step": round(1e3 * ms / w.iters, 2), "us_per_iter_marginal": round(us_iter, 2),
                         "gpairs_per_s": round((w.iters * w.n + w.n_test) / (ms * 1e-3) / 1e9, 4),
                         "cg_iters_per_s": round(w.iters / (ms * 1e-3), 1), "engine": engine,
                         "gpu_launches_per_step": launches, "floor_us": floor,
                         "frac_of_floor": (round(floor / us_iter, 4) if floor and us_iter > 0 else None)})
    # ---- the oracle on ONE host core ("also record a 1-core run for C1-C3"), and the
    #      explicit-K matvec at C1, the paper's baseline ("the standard matrix vector product with the
    #      kernel matrix"): fp64, baseline not target
    oracle_1core = []
    nthreads = O.num_threads()
    O.set_num_threads(1)
    try:
        for cfg, kname in (("C1", "kronecker"), ("C2", "kronecker"), ("C3", "symmetric")):
            w = synth.by_name(cfg)
            kernel = getattr(synth, kname.upper())
            Do = O.gram(w.base, w.Xd, gamma=w.gamma, coef0=w.coef0, degree=w.degree)
            To = None if w.Xt is None else O.gram(w.base, w.Xt, gamma=w.gamma, coef0=w.coef0, degree=w.degree)
            av = synth.random_vector(0, w.n)
            t0 = time.perf_counter()
            O.gvt_matvec(O.kernel_terms(kernel), Do, To, w.train_first, w.train_second, w.train_first,
                         w.train_second, av)
            dt = time.perf_counter() - t0
            rec = {"config": cfg, "kernel": kname, "matvec_s": round(dt, 4),
                   "gpairs_per_s": w.n / dt / 1e9, "cores": 1, "kind": "oracle per-term GVT (O4), fp64"}
            if cfg == "C1":
                t0 = time.perf_counter()
                O.explicit_matvec(kernel, Do, To, w.train_first, w.train_second, w.train_first, w.train_second, av)
                dte = time.perf_counter() - t0
                rec["explicit_K"] = {"matvec_s": round(dte, 5), "gpairs_per_s": w.n / dte / 1e9,
                                     "kind": "explicit kernel-matrix matvec (n x n kernel evaluations), fp64, 1 core"}
            oracle_1core.append(rec)
    finally:
        O.set_num_threads(nthreads)
    return {"runs": runs, "oracle_1core": oracle_1core,
            "note": "one B200; ms_per_step = Grams + fit(iters) + predict (graph-replayed solver); "
                    "us_per_iter_marginal = slope of the fit time from iters/2 to iters iterations; "
                    "frac_of_floor = SURVEY 8(d) floor per training matvec / us_per_iter_marginal"}


def max_over_ranks(v, world, args, dev):
    """Max of a per-rank device time over the ranks (NCCL: a CUDA tensor; gloo: a CPU tensor)."""
    if world <= 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=dev if args.comm == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2009_01054_b200 as G

    local_rank = local_rank % max(1, torch.cuda.device_count())  # --comm host: several ranks may share a GPU
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = workload(args.workload)
    kernel = G.KRONECKER if args.kernel is None else getattr(G, args.kernel.upper())
    if args.kernel is None:
        kernel = default_kernel(w)
    if kernel in G.HOMOGENEOUS_KERNELS and w.Xt is not None:
        w = synth.union_domain(w)
    terms = G.gvt_kernel_terms(kernel)
    ctx = G.Context(local_rank)
    ctx.set_option(G.OPT_ENGINE, args.engine)
    ctx.set_option(G.OPT_TC_PRECISION, 0 if args.precision == "fp16x3" else 1)
    ctx.set_option(G.OPT_EXCHANGE, args.exchange)
    ctx.set_option(G.OPT_SOLVER, G.SOLVER_MINRES if args.solver == "minres" else G.SOLVER_CG)
    ctx.set_option(G.OPT_CG_VARIANT, args.cg_variant)
    if world > 1 and args.comm == "host":
        ctx.comm_init_host(rank, world)   # host-mediated twin over the gloo group (ranks may share a GPU)
    elif world > 1:
        uid = G.gvt_nccl_unique_id() if rank == 0 else None
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        ctx.comm_init(obj[0], rank, world)

    # ---- shard (strong scaling: the whole workload is fixed as N grows; each rank generates the full workload
    #      and processes its drug range)
    f, s, y = w.train_first, w.train_second, w.y
    tf_, ts_ = w.test_first, w.test_second
    if world > 1:
        deg = np.bincount(f, minlength=w.m)
        bounds = G.gvt_partition(deg, world)
        lo, hi = bounds[rank], bounds[rank + 1]
        sel = (f >= lo) & (f < hi)
        f, s, y = f[sel], s[sel], y[sel]
        tsel = (tf_ >= lo) & (tf_ < hi)       # test pairs sharded by the same drug ranges
        tf_, ts_ = tf_[tsel], ts_[tsel]
    n_local, nt_local = len(f), len(tf_)

    def d(x):
        return torch.from_numpy(np.ascontiguousarray(x)).to(dev)

    Xd, Xt = d(w.Xd), (None if w.Xt is None else d(w.Xt))
    fD, sD, yD, tfD, tsD = d(f), d(s), d(y), d(tf_), d(ts_)
    m, q = w.m, w.q
    D = torch.empty((m, m), dtype=torch.float32, device=dev)
    T = None if Xt is None else torch.empty((q, q), dtype=torch.float32, device=dev)
    a = torch.empty(n_local, dtype=torch.float32, device=dev)
    scores = torch.empty(nt_local, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    phase_events = []  # per timed step: (start, grams done, fit done, predict done) on the launch stream

    def step(record=False):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if record else None
        if ev:
            ev[0].record(stream)
        ctx.gram(w.base, Xd, gamma=w.gamma, coef0=w.coef0, degree=w.degree, out=D)
        if T is not None:
            ctx.gram(w.base, Xt, gamma=w.gamma, coef0=w.coef0, degree=w.degree, out=T)
        if ev:
            ev[1].record(stream)
        _, it, _, _ = ctx.fit(D, T, fD, sD, yD, terms, w.lam, w.iters, 0.0, out=a, want_history=False)
        if ev:
            ev[2].record(stream)
        ctx.predict(D, T, tfD, tsD, fD, sD, a, terms, out=scores)
        if ev:
            ev[3].record(stream)
            phase_events.append(ev)
        return it

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    barrier()
    ctx.reset_stats()
    ctx.set_option(G.OPT_PROFILE, 1 if args.profile else 0)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            iters = step(record=True)
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    st = ctx.stats()
    ctx.set_option(G.OPT_PROFILE, 0)
    ms = max_over_ranks(ms, world, args, dev)
    ms_step = ms / args.steps
    pairs = float(iters) * w.n + w.n_test  # whole job
    # SURVEY 8(d) breakdown (this rank, CUDA events between the phases of each timed step): Grams,
    # fit (plan + iterations), predict (plan + stage 1 + stage 2)
    ph = np.array([[e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3])] for e in phase_events])
    gram_ms, fit_ms, pred_ms = (float(v) for v in ph.mean(axis=0))
    phases = {"gram_ms": gram_ms, "fit_ms": fit_ms, "predict_ms": pred_ms,
              "fit_gpairs_per_s": float(iters) * w.n / (fit_ms * 1e-3) / 1e9,
              "fit_cg_iters_per_s": float(iters) / (fit_ms * 1e-3),
              "predict_gpairs_per_s": w.n_test / (pred_ms * 1e-3) / 1e9,
              "note": "this rank's phase times; fit and predict include their plans (sorts, buckets)"}
    value = pairs / (ms_step * 1e-3) / 1e9

    # ---- standalone training matvec (Gpairs/s = n / t_matvec, median of 5 after 3
    #      warm-ups; each call includes its plan), on the fitted weights, outside the timed step
    matvec = None
    if world == 1:
        u = torch.empty(n_local, dtype=torch.float32, device=dev)
        for _ in range(3):
            ctx.matvec(D, T, fD, sD, fD, sD, a, terms, out=u)
        mv_ms = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.matvec(D, T, fD, sD, fD, sD, a, terms, out=u)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            mv_ms.append(e0.elapsed_time(e1))
        t = float(np.median(mv_ms))
        matvec = {"ms": t, "gpairs_per_s": w.n / (t * 1e-3) / 1e9, "runs": 5,
                  "note": "gvt_matvec over the training pairs (out = in sample), plan included, median of 5"}
        del u

    # ---- end to end through the C ABI with HOST buffers (pinned), copies inside the region
    e2e = None
    if not args.no_e2e:
        def pin(x):
            t = torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
            return t.numpy()
        hXd, hXt = pin(w.Xd), (None if w.Xt is None else pin(w.Xt))
        hf, hs, hy, htf, hts = pin(f), pin(s), pin(y), pin(tf_), pin(ts_)
        ha = pin(np.zeros(n_local, np.float32))
        hsc = pin(np.zeros(nt_local, np.float32))

        def step_host():
            ctx.gram(w.base, hXd, gamma=w.gamma, coef0=w.coef0, degree=w.degree, out=D)
            if T is not None:
                ctx.gram(w.base, hXt, gamma=w.gamma, coef0=w.coef0, degree=w.degree, out=T)
            ctx.fit(D, T, hf, hs, hy, terms, w.lam, w.iters, 0.0, out=ha, want_history=False)
            ctx.predict(D, T, htf, hts, hf, hs, ha, terms, out=hsc)

        step_host()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step_host()
        e1.record(stream)
        barrier()
        ems = max_over_ranks(e0.elapsed_time(e1), world, args, dev)
        h2d = (w.Xd.nbytes + (0 if w.Xt is None else w.Xt.nbytes) + 2 * (8 * n_local) + 4 * n_local +
               8 * nt_local + 4 * n_local) * world
        d2h = (4 * n_local + 4 * nt_local) * world
        e2e = {"value": pairs / (ems / args.steps * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": ems / args.steps}

    if rank != 0:
        return
    peaks = load_peaks()
    rl = roofline(st["kinds"], w, kernel, None, peaks, args.engine, args.precision) if args.profile else None
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        k, dt, cores = oracle_sample(w, kernel, n_targets=args.ref_targets, min_seconds=10.0)
        cpu = {"value": k / dt / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"fp64 oracle per-term GVT training matvec restricted to the outputs of {args.ref_targets} "
                         f"seeded targets, repeated for >= 10 s ({k} outputs in total; stage 1 streams all {w.n} "
                         f"pairs for those rows)",
               "seconds": round(dt, 2)}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(args, w, kernel, world),
            "runtime": {"last_engine": {1: "sparse", 2: "dense", 3: "single-CTA", 4: "persistent"}.get(st["last_engine"], None),
                        "exchange_used": {0: None, 1: "S-allgather", 2: "u-reduce"}.get(st.get("last_exchange", 0)),
                        "collectives": st["kinds"].get("collective", {}).get("count", 0)},
            "cg_iters_per_s": iters / (ms_step * 1e-3),
            "phases": phases,
            "matvec": matvec,
            "gpu_launches": int(st["launches"]),
            "kernel_ms": {k: round(v["ms"] / args.steps, 3) for k, v in st["kinds"].items()} if args.profile else None,
            "roofline": rl, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary()}
    if (args.gather_regime or args.configs) and world == 1:
        ctx.close()  # free the C5 workspaces first
        del D, T, a, scores, fD, sD, yD, tfD, tsD
        torch.cuda.empty_cache()
    if args.gather_regime and world == 1:
        line["gather_regime"] = gather_regime_leg(local_rank, peaks)
    if args.configs and world == 1:
        line["configs"] = configs_leg(local_rank)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--kernel", default=None)
    ap.add_argument("--engine", type=int, default=0)
    ap.add_argument("--precision", default="fp16x3", choices=["fp16x3", "tf32x3"])
    ap.add_argument("--exchange", type=int, default=2, choices=[0, 1, 2],
                    help="multi-GPU exchange per matvec: 0 = S slab all-gather, 1 = u reduce (NEXT-3), "
                         "2 = by estimated bytes (default)")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "host"],
                    help="N > 1: NCCL (one rank per GPU) or the library's host-mediated twin over gloo (ranks may "
                         "share a GPU; a test of the launcher and the data-parallel path on a one-GPU box)")
    ap.add_argument("--solver", default="cg", choices=["cg", "minres"])
    ap.add_argument("--cg-variant", type=int, default=0, choices=[0, 1],
                    help="0 = Hestenes-Stiefel CG, 1 = Chronopoulos-Gear (one reduction per iteration)")
    ap.add_argument("--no-profile", dest="profile", action="store_false")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gather-regime", dest="gather_regime", action="store_false",
                    help="skip the sparse-engine gather-regime leg (0.2 %% density at C5 object counts)")
    ap.add_argument("--no-configs", dest="configs", action="store_false",
                    help="skip the per-config legs (C1-C4 every kernel, oracle 1-core C1-C3, explicit-K C1)")
    ap.add_argument("--ref-targets", type=int, default=8,
                    help="oracle sample per step: the outputs of this many seeded targets (cpu_baseline and "
                         "--impl reference)")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `bench.py --gpus N` outside a launcher: re-run this command under torch.distributed.run, one
        # rank per GPU (the driver's own launch sets WORLD_SIZE and lands below directly)
        import socket
        sock = socket.socket()
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
        sock.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        # never time one world size and report another
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.comm == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")   # the "nranks N" init lines, for the driver's check
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    try:
        run_gpu(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
