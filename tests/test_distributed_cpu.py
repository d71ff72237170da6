"""Multi-process (world_size 2, gloo, CPU) checks of the data-parallel decomposition
 -- no GPU needed.

Each rank holds a drug-range shard of the training pairs (gvt_partition), gathers the
in-sample and p over the ranks, runs GVT stage 1 on its own X-row slab (gvt_slab_bounds,
the same host function the CUDA engine uses), all-gathers the equal-width S slabs, runs
stage 2 on its own outputs and all-reduces the CG dot products.  The stages are fp64 numpy
models of the library's kernels; what is under test is the partition/slab/gather logic:
the sharded CG must reproduce the single-process oracle CG on the same data.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as tmp  # noqa: E402

import oracle as O  # noqa: E402
import paper_2009_01054_b200 as G  # noqa: E402
import synth  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _all_gather_var(x, world):
    """variable-length all-gather in rank order (pads to the max length)"""
    n = torch.tensor([len(x)], dtype=torch.int64)
    ns = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(ns, n)
    ns = [int(v.item()) for v in ns]
    nmax = max(ns)
    buf = torch.zeros(nmax, dtype=torch.float64)
    buf[: len(x)] = torch.from_numpy(np.asarray(x, dtype=np.float64))
    out = [torch.zeros(nmax, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(out, buf)
    return np.concatenate([o.numpy()[:k] for o, k in zip(out, ns)]), ns


def _worker(rank, world, port, iters, ret, exchange=0):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = synth.config1()
        D = O.gram(w.base, w.Xd, gamma=w.gamma)
        T = O.gram(w.base, w.Xt, gamma=w.gamma)
        m, q = w.m, w.q
        f, s, y = w.train_first, w.train_second, w.y.astype(np.float64)
        # ---- drug-range shards (library host logic)
        bounds = G.gvt_partition(np.bincount(f, minlength=m), world)
        mine = (f >= bounds[rank]) & (f < bounds[rank + 1])
        lf, ls, ly = f[mine], s[mine], y[mine]
        # ---- gathered in-sample (rank order) and the X-row slabs of the Kronecker group
        ff, counts = _all_gather_var(lf, world)
        fs, _ = _all_gather_var(ls, world)
        ff, fs = ff.astype(np.int64), fs.astype(np.int64)
        row_ptr = np.concatenate([[0], np.cumsum(np.bincount(ff, minlength=m))])
        sb = G.gvt_slab_bounds(row_ptr, world)
        W = int(-(-max(np.diff(sb).max(), 1) // 32) * 32)
        lo, hi = int(sb[rank]), int(sb[rank + 1])

        offs = np.concatenate([[0], np.cumsum(counts)])

        def matvec_u(p_local):
            """u-exchange (GVT_OPT_EXCHANGE = 1, NEXT-3): stage 2 of this rank's slab for EVERY
            output (the gathered sample), then each output segment goes to its owner, which sums
            the ranks' contributions in rank order (the library's send/recv + rank-order sum: the
            bytes of a variable-count reduce-scatter, 4 n instead of 4 q m, with a fixed order)."""
            p_full, _ = _all_gather_var(p_local, world)
            B = np.zeros((hi - lo, q))
            sel = (ff >= lo) & (ff < hi)
            np.add.at(B, (ff[sel] - lo, fs[sel]), p_full[sel])
            S_slab = T @ B.T                                   # q x (hi - lo)
            partial = np.einsum("ih,ih->i", D[ff][:, lo:hi], S_slab[fs])
            recv = [None] * world
            for g in range(world):                             # segment g travels to its owner g
                seg = torch.from_numpy(np.ascontiguousarray(partial[offs[g]:offs[g + 1]]))
                parts = [torch.zeros_like(seg) for _ in range(world)] if g == rank else None
                dist.gather(seg, parts, dst=g)
                if g == rank:
                    recv = [t.numpy() for t in parts]
            local = np.zeros(int(counts[rank]))
            for g in range(world):                             # rank-order sum
                local = local + recv[g]
            return local

        def matvec(p_local):
            if exchange == 1:
                return matvec_u(p_local)
            p_full, _ = _all_gather_var(p_local, world)
            # stage 1 on this rank's slab: S[:, h] for h in [lo, hi)
            B = np.zeros((hi - lo, q))
            sel = (ff >= lo) & (ff < hi)
            np.add.at(B, (ff[sel] - lo, fs[sel]), p_full[sel])
            slab = np.zeros((q, W))
            slab[:, : hi - lo] = T @ B.T
            # all-gather the equal-width slabs
            outs = [torch.zeros(q * W, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(outs, torch.from_numpy(slab.reshape(-1)))
            S = np.zeros((q, m))
            for g in range(world):
                a, b = int(sb[g]), int(sb[g + 1])
                S[:, a:b] = outs[g].numpy().reshape(q, W)[:, : b - a]
            # stage 2 on this rank's outputs
            return np.einsum("ih,ih->i", D[lf], S[ls])

        def dot(a, b):
            t = torch.tensor([float(a @ b)], dtype=torch.float64)
            dist.all_reduce(t)
            return float(t.item())

        x = np.zeros_like(ly)
        r = ly.copy()
        p = r.copy()
        rho = dot(r, r)
        for _ in range(iters):
            Ap = matvec(p) + w.lam * p
            alpha = rho / dot(p, Ap)
            x += alpha * p
            r -= alpha * Ap
            rho1 = dot(r, r)
            p = r + (rho1 / rho) * p
            rho = rho1
        xs, _ = _all_gather_var(x, world)
        if rank == 0:
            order = np.concatenate([np.nonzero((f >= bounds[g]) & (f < bounds[g + 1]))[0] for g in range(world)])
            full = np.empty_like(xs)
            full[order] = xs
            ret.put((full, [int(v) for v in sb], [int(v) for v in bounds], counts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange", [0, 1], ids=["S-allgather", "u-reduce"])
@pytest.mark.parametrize("world", [2])
def test_sharded_cg_equals_single_process_oracle(world, exchange):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    iters = 12
    tmp.start_processes(_worker, args=(world, _free_port(), iters, q, exchange), nprocs=world, join=True,
                        start_method="spawn")
    a_sharded, sb, bounds, counts = q.get(timeout=60)
    w = synth.config1()
    D = O.gram(w.base, w.Xd, gamma=w.gamma)
    T = O.gram(w.base, w.Xt, gamma=w.gamma)
    a_ref, _, _, _ = O.cg(O.kernel_terms(O.KRONECKER), D, T, w.train_first, w.train_second, w.y, w.lam, iters)
    # fp64 on both sides; only the summation order differs (a wrong partition is O(1) off)
    assert np.linalg.norm(a_sharded - a_ref) / np.linalg.norm(a_ref) < 1e-8
    assert sb[0] == 0 and sb[-1] == w.m and all(b % 32 == 0 for b in sb[1:-1])
    assert sum(counts) == w.n and bounds[0] == 0 and bounds[-1] == w.m


def test_slab_bounds_definition():
    rng = np.random.default_rng(0)
    for nrow, G_ in [(1, 1), (40, 2), (1000, 3), (20000, 8), (5, 8)]:
        rp = np.concatenate([[0], np.cumsum(rng.integers(0, 50, nrow))])
        b = G.gvt_slab_bounds(rp, G_)
        E = rp[-1]
        ref = [0]
        for s in range(1, G_):
            h = int(np.searchsorted(rp, int(E * s / G_), side="left"))
            h = min(max(-(-h // 32) * 32, ref[-1]), nrow)
            ref.append(h)
        ref.append(nrow)
        assert list(b) == ref


def test_slab_bounds_cost_definition():
    """gvt_slab_bounds_cost: bounds[s] = the first row h whose cost w_e * rp[h] + w_r * h reaches the
    s/G quantile, rounded up to 32, monotone; w_r = 0 reproduces gvt_slab_bounds."""
    rng = np.random.default_rng(1)
    for nrow, G_ in [(1, 1), (40, 2), (1000, 3), (20000, 8), (5, 8)]:
        rp = np.concatenate([[0], np.cumsum(rng.integers(0, 50, nrow))])
        assert list(G.gvt_slab_bounds_cost(rp, G_, 1.0, 0.0)) == list(G.gvt_slab_bounds(rp, G_))
        for we, wr in [(0.0, 1.0), (1.0, 3.0), (0.25, 100.0)]:
            b = G.gvt_slab_bounds_cost(rp, G_, we, wr)
            cost = we * rp + wr * np.arange(nrow + 1)
            ref = [0]
            for s_ in range(1, G_):
                h = int(np.argmax(cost >= cost[-1] * s_ / G_)) if cost[-1] > 0 else 0
                ref.append(min(max(-(-h // 32) * 32, ref[-1]), nrow))
            ref.append(nrow)
            assert list(b) == ref, (nrow, G_, we, wr)


def test_dense_slabs_balanced_on_degree_sorted_c5_shape():
    """ADVICE r1 / VERDICT r1 item 4: with drug ids ordered by degree (C5's capped Zipf(1.1) degrees,
    1e8 pairs over 20000 drugs), entry-balanced slabs give the dense engine (whose GEMM cost is the
    slab's ROWS) rows max/mean ~3.2 at 8 slabs; the engine's dense weights (0, 1) give <= 1.1."""
    deg = np.sort(synth.zipf_degrees(20_000, 100_000_000, 20_000))[::-1]
    rp = np.concatenate([[0], np.cumsum(deg)])
    by_entries = np.diff(G.gvt_slab_bounds(rp, 8))
    by_rows = np.diff(G.gvt_slab_bounds_cost(rp, 8, 0.0, 1.0))
    assert by_entries.max() / by_entries.mean() > 3.0
    assert by_rows.max() / by_rows.mean() <= 1.1
    # the sparse weights balance the estimated cost (entries x q_out plus rows x 4 n / 6.4e6 under the
    # u-exchange) to within one 32-row rounding step of the cost
    we, wr = 20_000 / 3.3e6, 4.0 * 1e8 / 6.4e6
    b = G.gvt_slab_bounds_cost(rp, 8, we, wr)
    cost = we * np.diff(rp[b]) + wr * np.diff(b)
    assert cost.max() / cost.mean() <= 1.1


def test_bench_rejects_mismatched_world():
    """bench.py never times one world size and reports another: --gpus 2 under WORLD_SIZE=1 exits 2
    (before touching a GPU)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--workload", "C1"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr
