"""Seeded synthetic workloads C1..C5 (and tiny random instances) for the GVT hot path.

This module is the ONLY code shared by the oracle side (``oracle/``, tests) and the
CUDA side (``paper_2009_01054_b200``, bench).  It draws random numbers and lays out
index arrays; it contains none of the method's arithmetic (no Gram, no kernel, no
GVT, no solver).  Every recipe follows SURVEY.md §8(d) (the stand-ins for the
paper's datasets, Table 5 at PAPER.md:777-785) and the readings
S5-S11 recorded in DESIGN.md.

All draws use ``numpy.random.default_rng(seed)`` (PCG64) with seed = config number,
in the order listed in each generator.  Pairs are int32, features / labels float32.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

# Kernel names (mirror include/gvt.h enum gvt_kernel; plain integers, no arithmetic).
LINEAR, POLY2D, GAUSSIAN, KRONECKER, SYMMETRIC, ANTISYMMETRIC, RANKING, MLPK, CARTESIAN = range(9)
KERNEL_NAMES = ["linear", "poly2d", "gaussian", "kronecker", "symmetric",
                "antisymmetric", "ranking", "mlpk", "cartesian"]
HOMOGENEOUS_KERNELS = (SYMMETRIC, ANTISYMMETRIC, RANKING, MLPK)

# Base kernels (mirror enum gvt_base).
BASE_LINEAR, BASE_GAUSSIAN, BASE_POLY, BASE_TANIMOTO = range(4)


@dataclasses.dataclass
class Workload:
    """One synthetic problem.  ``Xd``/``Xt`` are object features; ``Xt is None`` means
    homogeneous (one object table)."""
    name: str
    Xd: np.ndarray                      # (m, dim) float32
    Xt: Optional[np.ndarray]            # (q, dim) float32 or None (homogeneous)
    base: int                           # BASE_LINEAR / BASE_GAUSSIAN / BASE_POLY
    gamma: float
    train_first: np.ndarray             # (n,) int32
    train_second: np.ndarray            # (n,) int32
    y: np.ndarray                       # (n,) float32
    test_first: np.ndarray              # (n_hat,) int32
    test_second: np.ndarray             # (n_hat,) int32
    lam: float
    iters: int
    kernels: tuple                      # pairwise kernels this config runs
    coef0: float = 1.0
    degree: int = 2

    @property
    def m(self) -> int:
        return int(self.Xd.shape[0])

    @property
    def q(self) -> int:
        return int(self.Xd.shape[0] if self.Xt is None else self.Xt.shape[0])

    @property
    def n(self) -> int:
        return int(self.train_first.shape[0])

    @property
    def n_test(self) -> int:
        return int(self.test_first.shape[0])


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


# --------------------------------------------------------------------------- C1
def config1() -> Workload:
    """C1 tiny Kronecker KRR (BASELINE.json configs[0]): m=40, q=60, dim 16 N(0,1),
    Gaussian gamma=1/16; 1500 distinct grid cells, first 1000 train, next 500 test
    (S11); y ~ N(0,1); lambda=1; 50 CG iterations."""
    rng = np.random.default_rng(1)
    Xd = rng.standard_normal((40, 16), dtype=np.float32)
    Xt = rng.standard_normal((60, 16), dtype=np.float32)
    cells = rng.choice(40 * 60, 1500, replace=False)
    y = rng.standard_normal(1000, dtype=np.float32)
    d, t = cells // 60, cells % 60
    return Workload("C1", Xd, Xt, BASE_GAUSSIAN, 1.0 / 16, _i32(d[:1000]), _i32(t[:1000]), _f32(y),
                    _i32(d[1000:]), _i32(t[1000:]), 1.0, 50, (KRONECKER,))


# --------------------------------------------------------------------------- C2
def config2() -> Workload:
    """C2 complete-grid drug-target Kronecker KRR (configs[1]): m=68, q=442, all 30 056
    cells d-major, linear base kernel on dim-256 N(0,1) features; y = x_d^T W x_t + eps,
    W_ij ~ N(0,1)/256, eps ~ N(0, 0.1^2) (S9); lambda=1e-2; 100 CG iterations.
    The label recipe draws W and eps here: it is data synthesis, not the method."""
    rng = np.random.default_rng(2)
    Xd = rng.standard_normal((68, 256), dtype=np.float32)
    Xt = rng.standard_normal((442, 256), dtype=np.float32)
    W = rng.standard_normal((256, 256)) / 256.0
    eps = rng.normal(0.0, 0.1, size=68 * 442)
    d = np.repeat(np.arange(68), 442)
    t = np.tile(np.arange(442), 68)
    y = np.einsum("ij,jk,ik->i", Xd[d].astype(np.float64), W, Xt[t].astype(np.float64)) + eps
    return Workload("C2", Xd, Xt, BASE_LINEAR, 0.0, _i32(d), _i32(t), _f32(y),
                    _i32(d), _i32(t), 1e-2, 100, (KRONECKER,))


def _unrank_upper(idx: np.ndarray, m: int):
    """Map linear indices of the strict upper triangle (row-major, i<j) of an m x m grid to (i, j)."""
    idx = idx.astype(np.int64)
    # row i starts at offset i*m - i*(i+1)/2 ; solve for i with float then fix up.
    i = np.floor((2 * m - 1 - np.sqrt((2 * m - 1) ** 2 - 8.0 * idx)) / 2).astype(np.int64)
    start = i * m - i * (i + 1) // 2
    over = idx < start
    i[over] -= 1
    start = i * m - i * (i + 1) // 2
    nxt = (i + 1) * m - (i + 1) * (i + 2) // 2
    under = idx >= nxt
    i[under] += 1
    start = i * m - i * (i + 1) // 2
    j = idx - start + i + 1
    return i, j


# --------------------------------------------------------------------------- C3
def config3(n: int = 200_000, n_test: int = 100_000) -> Workload:
    """C3 homogeneous protein-protein (configs[2]): 2000 objects, dim 128 N(0,1),
    Gaussian gamma=1/128 (S5); n distinct unordered i<j pairs (10% of the triangle);
    y = +-1 uniform; lambda=1 (S8); 100 CG iterations; optional further distinct test
    pairs (S11).  Kernels: Symmetric, Anti-symmetric, Cartesian."""
    rng = np.random.default_rng(3)
    m = 2000
    X = rng.standard_normal((m, 128), dtype=np.float32)
    tri = m * (m - 1) // 2
    cells = rng.choice(tri, n + n_test, replace=False)
    y = rng.choice(np.array([-1.0, 1.0], dtype=np.float32), size=n)
    i, j = _unrank_upper(cells, m)
    return Workload("C3", X, None, BASE_GAUSSIAN, 1.0 / 128, _i32(i[:n]), _i32(j[:n]), _f32(y),
                    _i32(i[n:]), _i32(j[n:]), 1.0, 100, (SYMMETRIC, ANTISYMMETRIC, CARTESIAN))


# --------------------------------------------------------------------------- C4
def config4(n: int = 2_000_000, n_test: int = 1_000_000) -> Workload:
    """C4 multi-term kernels (configs[3]): 5000 drugs x 3000 targets, dim 64 N(0,1),
    Gaussian gamma=1/64 (S6); n train + n_test distinct cells (13.3% density);
    y ~ N(0,1) (S10); lambda=1; 50 CG iterations.  Kernels Poly2D (heterogeneous) and
    MLPK / Ranking on the union-domain reading S7 (see ``union_domain``)."""
    rng = np.random.default_rng(4)
    Xd = rng.standard_normal((5000, 64), dtype=np.float32)
    Xt = rng.standard_normal((3000, 64), dtype=np.float32)
    cells = rng.choice(5000 * 3000, n + n_test, replace=False)
    y = rng.standard_normal(n, dtype=np.float32)
    d, t = cells // 3000, cells % 3000
    return Workload("C4", Xd, Xt, BASE_GAUSSIAN, 1.0 / 64, _i32(d[:n]), _i32(t[:n]), _f32(y),
                    _i32(d[n:]), _i32(t[n:]), 1.0, 50, (POLY2D, MLPK, RANKING))


def union_domain(w: Workload) -> Workload:
    """Reading S7: one object table of m+q objects (drugs 0..m-1, targets m..m+q-1);
    pair (d, t) becomes (d, m+t).  Used to run homogeneous kernels on C4."""
    assert w.Xt is not None
    X = np.ascontiguousarray(np.concatenate([w.Xd, w.Xt], axis=0))
    off = np.int32(w.m)
    return dataclasses.replace(w, name=w.name + "-union", Xd=X, Xt=None,
                               train_second=_i32(w.train_second + off),
                               test_second=_i32(w.test_second + off))


# --------------------------------------------------------------------------- C5
def zipf_degrees(m: int, n: int, cap: int, s: float = 1.1) -> np.ndarray:
    """Capped Zipf degrees deg_k = min(cap, c*k^-s), k=1..m, with c found by bisection so
    the real-valued degrees sum to n, integerised by largest remainder to sum exactly n."""
    k = np.arange(1, m + 1, dtype=np.float64)
    base = k ** (-s)
    lo, hi = 0.0, float(n) * 10
    for _ in range(200):
        c = 0.5 * (lo + hi)
        tot = np.minimum(cap, c * base).sum()
        if tot < n:
            lo = c
        else:
            hi = c
    real = np.minimum(cap, hi * base)
    deg = np.floor(real).astype(np.int64)
    rem = n - int(deg.sum())
    frac = real - deg
    frac[deg >= cap] = -1.0
    if rem > 0:
        order = np.argsort(-frac, kind="stable")[:rem]
        deg[order] += 1
    return deg


def _disk_cached(fn):
    """With GVT_SYNTH_CACHE=<dir>, keep generated workloads as .npz files keyed by the call's
    arguments (the C5 draw takes ~20 s; measurement scripts regenerate it per process).  The
    arrays are the generator's own output, saved and reloaded unchanged."""
    import functools
    import os

    @functools.wraps(fn)
    def wrapper(*args, **kw):
        d = os.environ.get("GVT_SYNTH_CACHE")
        if not d:
            return fn(*args, **kw)
        key = fn.__name__ + "_" + "_".join(map(str, args)) + "_" + "_".join(f"{k}{v}" for k, v in sorted(kw.items()))
        path = os.path.join(d, key + ".npz")
        fields = [f.name for f in dataclasses.fields(Workload)]
        if os.path.exists(path):
            z = np.load(path, allow_pickle=True)
            vals = {f: (z[f].item() if z[f].dtype == object else z[f]) for f in fields}
            vals["kernels"] = tuple(int(k) for k in z["kernels"])
            return Workload(**vals)
        w = fn(*args, **kw)
        os.makedirs(d, exist_ok=True)
        arrs = {f: getattr(w, f) for f in fields}
        arrs = {k: (np.array(v, dtype=object) if v is None or isinstance(v, (str, float, int)) else np.asarray(v))
                for k, v in arrs.items()}
        tmp = path + ".tmp.npz"
        np.savez(tmp, **arrs)
        os.replace(tmp, path)
        return w
    return wrapper


@_disk_cached
def config5(n: int = 100_000_000, n_test: int = 20_000_000, m: int = 20_000, dim: int = 128,
            chunk: int = 512) -> Workload:
    """C5 large-scale Kronecker KRR (configs[4]): m=q=20000, dim 128 N(0,1), Gaussian
    gamma=1/128 (S5); n = 1e8 train pairs with capped Zipf(1.1) drug degrees (cap = q),
    drug ranks permuted onto ids, each drug drawing deg distinct targets by weighted
    sampling without replacement (Efraimidis-Spirakis keys log(u)/w, target weights
    proportional to rank^-1.1 permuted onto ids); pair order is a seeded shuffle;
    n_test i.i.d. test pairs with d ~ degree and t ~ target weight (S11); y ~ N(0,1);
    lambda = 1; 30 CG iterations.  ``n``/``m`` can be reduced for scaled-down tests."""
    q = m
    rng = np.random.default_rng(5)
    Xd = rng.standard_normal((m, dim), dtype=np.float32)
    Xt = rng.standard_normal((q, dim), dtype=np.float32)
    deg_by_rank = zipf_degrees(m, n, q)
    drug_perm = rng.permutation(m)            # rank r -> drug id drug_perm[r]
    deg = np.empty(m, dtype=np.int64)
    deg[drug_perm] = deg_by_rank
    tw_by_rank = np.arange(1, q + 1, dtype=np.float64) ** (-1.1)
    target_perm = rng.permutation(q)
    tw = np.empty(q, dtype=np.float64)
    tw[target_perm] = tw_by_rank
    inv_w = 1.0 / tw
    first = np.empty(n, dtype=np.int32)
    second = np.empty(n, dtype=np.int32)
    pos = 0
    for d0 in range(0, m, chunk):
        d1 = min(m, d0 + chunk)
        u = rng.random((d1 - d0, q))
        keys = np.log(u) * inv_w                   # larger is better (closer to 0)
        for r in range(d1 - d0):
            k = int(deg[d0 + r])
            if k == 0:
                continue
            if k >= q:
                sel = np.arange(q)
            else:
                sel = np.sort(np.argpartition(-keys[r], k - 1)[:k])
            first[pos:pos + k] = d0 + r
            second[pos:pos + k] = sel
            pos += k
    assert pos == n
    order = rng.permutation(n)
    first = first[order]
    second = second[order]
    y = rng.standard_normal(n, dtype=np.float32)
    pd = deg / deg.sum()
    pt = tw / tw.sum()
    tf = rng.choice(m, size=n_test, p=pd)
    ts = rng.choice(q, size=n_test, p=pt)
    return Workload("C5", Xd, Xt, BASE_GAUSSIAN, 1.0 / dim, _i32(first), _i32(second), _f32(y),
                    _i32(tf), _i32(ts), 1.0, 30, (KRONECKER,))


def gather_regime(m: int = 20_000, n: int = 800_000, n_test: int = 2_000_000, dim: int = 128,
                  seed: int = 7) -> Workload:
    """The SIMT-gather regime at C5 object counts (density below ~2 %, where the
    north star's "stage-2 gather at >= 60 % of HBM" applies): m = q objects, dim N(0,1)
    features, Gaussian gamma = 1/dim (S5); n uniform training pairs (default 0.2 % of the grid,
    Heterodimer-like), n_test uniform test pairs, y ~ N(0,1); lambda 1, 30 iterations."""
    rng = np.random.default_rng(seed)
    Xd = rng.standard_normal((m, dim), dtype=np.float32)
    Xt = rng.standard_normal((m, dim), dtype=np.float32)
    f = rng.integers(0, m, n)
    s = rng.integers(0, m, n)
    tf = rng.integers(0, m, n_test)
    ts = rng.integers(0, m, n_test)
    y = rng.standard_normal(n, dtype=np.float32)
    return Workload("gather", Xd, Xt, BASE_GAUSSIAN, 1.0 / dim, _i32(f), _i32(s), _f32(y), _i32(tf), _i32(ts),
                    1.0, 30, (KRONECKER,))


CONFIGS = {"C1": config1, "C2": config2, "C3": config3, "C4": config4, "C5": config5}


def by_name(name: str, **kw) -> Workload:
    return CONFIGS[name](**kw)


# --------------------------------------------------------------------------- tiny instances
def tiny(seed: int, m: int = 5, q: int = 4, n: int = 12, n_out: int = 9, dim: int = 3,
         homogeneous: bool = False, duplicates: bool = True, self_pairs: bool = True) -> Workload:
    """Tiny random instance for brute-force pins: pairs drawn WITH replacement (so
    duplicates occur, S17), self pairs allowed in the homogeneous case (S18),
    out-sample different from in-sample."""
    rng = np.random.default_rng(10_000 + seed)
    Xd = rng.standard_normal((m, dim), dtype=np.float32)
    Xt = None if homogeneous else rng.standard_normal((q, dim), dtype=np.float32)
    qq = m if homogeneous else q
    f = rng.integers(0, m, n)
    s = rng.integers(0, qq, n)
    if not self_pairs and homogeneous:
        s = np.where(s == f, (s + 1) % m, s)
    if not duplicates:
        cells = rng.choice(m * qq, min(n, m * qq), replace=False)
        f, s = cells // qq, cells % qq
    of = rng.integers(0, m, n_out)
    os_ = rng.integers(0, qq, n_out)
    y = rng.standard_normal(len(f)).astype(np.float32)
    return Workload(f"tiny{seed}", Xd, Xt, BASE_GAUSSIAN, 0.5, _i32(f), _i32(s), _f32(y),
                    _i32(of), _i32(os_), 1.0, 10, (KRONECKER,))


def parity_grid(pattern: str, m: int, q: int, seed: int = 0, val_frac: float = 0.25):
    """The paper's toy problems (Figure 1; SPEC.md generate_synthetic):
    'chessboard' y(d,t) = parity(d) XOR parity(t), 'tablecloth' y(d,t) = 1 iff
    parity(d) + parity(t) >= 1; features [1, parity] for drugs and targets (the constant
    feature spans bias, marginals and interaction).  All m x q cells, randomly split
    (seeded) into an inner training sample and a validation sample (Setting 1).
    Returns (Workload with the linear base kernel, validation labels); labels are 0/1."""
    if pattern not in ("chessboard", "tablecloth"):
        raise ValueError(pattern)
    rng = np.random.default_rng(40_000 + seed)
    pd, pt = np.arange(m) % 2, np.arange(q) % 2
    Xd = np.stack([np.ones(m), pd], 1)
    Xt = np.stack([np.ones(q), pt], 1)
    cells = rng.permutation(m * q)
    d, t = cells // q, cells % q
    lab = (pd[d] ^ pt[t]) if pattern == "chessboard" else ((pd[d] + pt[t]) >= 1).astype(np.int64)
    n_val = int(round(val_frac * m * q))
    w = Workload(f"{pattern}{m}x{q}", _f32(Xd), _f32(Xt), BASE_LINEAR, 1.0, _i32(d[n_val:]), _i32(t[n_val:]),
                 _f32(lab[n_val:]), _i32(d[:n_val]), _i32(t[:n_val]), 1e-5, 100, (KRONECKER,))
    return w, _f32(lab[:n_val])


def kernel_filling(n_pairs: int, seed: int = 0, n_objects: int = 2967, dim: int = 1024, n_clusters: int = 24,
                   flip: float = 0.2, label_noise: float = 0.05, val_frac: float = 0.25):
    """Stand-in for the paper's kernel-filling data set (Table 5: 2967 drugs,
    complete homogeneous grid), whose real drug kernels are not in the container.
    Objects: n_objects binary fingerprints of length dim, each a copy of one of n_clusters random
    prototypes (density 10 %) with every bit flipped with probability `flip` -- Tanimoto
    similarity then tracks cluster membership.  Labels: 1 if the two objects share a cluster,
    else 0, each flipped with probability `label_noise` (a planted, noisy pairwise structure; no
    method arithmetic).  Pairs: as in the paper, a
    subset of k objects with k(k-1)/2 ~ n_pairs gives all its unordered pairs i < j, shuffled and
    split 75 % inner training / 25 % validation (Setting 1).  Returns (Workload with the Tanimoto
    base kernel and homogeneous ids, validation labels); training labels are in w.y."""
    rng = np.random.default_rng(50_000 + seed)
    protos = rng.uniform(size=(n_clusters, dim)) < 0.10
    cl = rng.integers(0, n_clusters, n_objects)
    X = protos[cl] ^ (rng.uniform(size=(n_objects, dim)) < flip)
    k = int(min(n_objects, max(2, round((1 + math.sqrt(1 + 8 * n_pairs)) / 2))))
    sub = np.sort(rng.choice(n_objects, k, replace=False))
    iu, ju = np.triu_indices(k, 1)
    order = rng.permutation(len(iu))
    f, s = sub[iu[order]], sub[ju[order]]
    lab = ((cl[f] == cl[s]) ^ (rng.uniform(size=len(f)) < label_noise)).astype(np.float32)
    n_val = int(round(val_frac * len(f)))
    w = Workload(f"kf{len(f)}", _f32(X), None, BASE_TANIMOTO, 1.0, _i32(f[n_val:]), _i32(s[n_val:]),
                 _f32(lab[n_val:]), _i32(f[:n_val]), _i32(s[:n_val]), 1e-5, 300,
                 (LINEAR, POLY2D, KRONECKER, CARTESIAN, SYMMETRIC, MLPK))
    return w, _f32(lab[:n_val])


def random_vector(seed: int, n: int) -> np.ndarray:
    """Seeded N(0,1) float32 vector (the 'a' of a standalone matvec)."""
    return np.random.default_rng(20_000 + seed).standard_normal(n, dtype=np.float32)


def sample_indices(seed: int, n: int, k: int) -> np.ndarray:
    """Seeded sample of k distinct output positions in [0, n) (sorted), for sampled parity."""
    k = min(k, n)
    return np.sort(np.random.default_rng(30_000 + seed).choice(n, k, replace=False)).astype(np.int64)
