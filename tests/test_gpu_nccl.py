"""The NCCL data plane executed on one GPU (-m gpu): gvt_comm_init with a unique id and world 1
creates a one-rank NCCL communicator, and the library then runs its data-parallel path with its
real NCCL calls -- the in-sample id / p gathers (grouped ncclBroadcast), the S slab all-gather
(ncclAllGather, captured into the solver's CUDA graph), the solver's fp64 partial all-gathers,
the u-exchange (ncclSend / ncclRecv to the segment owners + ncclAllGather of MLPK's tail) and
the plan-time count all-gathers.

Checks: every call issued collectives (the "collective" counter of gvt_get_stats); the results
equal the single-GPU path's bit for bit (one rank: the exchanges are copies and the rank-order
sums are over one rank), and the fits match the fp64 oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import paper_2009_01054_b200 as G  # noqa: E402
import synth  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def rel(x, ref):
    x, ref = np.asarray(x, np.float64), np.asarray(ref, np.float64)
    return np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-30)


@pytest.fixture(scope="module")
def pair():
    torch.cuda.set_device(0)
    nc = G.Context(0)
    nc.comm_init(G.gvt_nccl_unique_id(), 0, 1)  # one-rank NCCL communicator
    plain = G.Context(0)
    for c in (nc, plain):
        c.set_option(G.OPT_COMPACT, 0)  # compaction is single-GPU only; keep the paths comparable
    yield nc, plain
    nc.close()
    plain.close()


def _collectives(ctx):
    return ctx.stats()["kinds"].get("collective", {}).get("count", 0)


def _workload(kernel):
    return synth.config1() if kernel == G.KRONECKER else synth.config3(n=20_000, n_test=3_000)


CASES = [  # (kernel, engine, exchange, solver: 0 CG, 1 MINRES, 2 single-reduction CG)
    (G.KRONECKER, G.ENGINE_DENSE, 0, 0), (G.KRONECKER, G.ENGINE_SPARSE, 0, 0), (G.KRONECKER, G.ENGINE_DENSE, 1, 0),
    (G.KRONECKER, G.ENGINE_DENSE, 0, 1), (G.KRONECKER, G.ENGINE_DENSE, 0, 2), (G.SYMMETRIC, G.ENGINE_AUTO, 0, 0),
    (G.SYMMETRIC, G.ENGINE_SPARSE, 1, 0), (G.MLPK, G.ENGINE_DENSE, 1, 0), (G.MLPK, G.ENGINE_SPARSE, 0, 0),
]


@pytest.mark.parametrize("case", CASES, ids=[f"k{k}-e{e}-x{x}-s{s}" for k, e, x, s in CASES])
def test_nccl_world1_fit_predict_matvec(pair, case):
    kernel, engine, exchange, solver = case
    nc, plain = pair
    w = _workload(kernel)
    terms = G.gvt_kernel_terms(kernel)
    outs = []
    for c in (nc, plain):
        c.set_option(G.OPT_ENGINE, engine)
        c.set_option(G.OPT_EXCHANGE, exchange)
        c.set_option(G.OPT_SOLVER, 1 if solver == 1 else 0)
        c.set_option(G.OPT_CG_VARIANT, 1 if solver == 2 else 0)
        c.reset_stats()
        D = c.gram(w.base, dev(w.Xd), gamma=w.gamma)
        T = None if w.Xt is None else c.gram(w.base, dev(w.Xt), gamma=w.gamma)
        f, s = dev(w.train_first), dev(w.train_second)
        a, it, hist, code = c.fit(D, T, f, s, dev(w.y), terms, w.lam, 20)  # graph-replayed iterations
        sc = c.predict(D, T, dev(w.test_first), dev(w.test_second), f, s, a, terms)
        u = c.matvec(D, T, f, s, f, s, dev(synth.random_vector(3, w.n)), terms)
        torch.cuda.synchronize()
        outs.append((a.cpu().numpy(), sc.cpu().numpy(), u.cpu().numpy(), it, hist, _collectives(c)))
        c.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)
        c.set_option(G.OPT_EXCHANGE, 0)
        c.set_option(G.OPT_SOLVER, 0)
        c.set_option(G.OPT_CG_VARIANT, 0)
    (a1, sc1, u1, it1, h1, n1), (a0, sc0, u0, it0, h0, n0) = outs
    assert n1 > 20, "the NCCL context issued no collectives per iteration"
    assert n0 == 0
    assert it1 == it0 == 20
    # one rank: exchanges are copies, rank-order sums run over one rank -> the same bits
    assert np.array_equal(a1, a0) and np.array_equal(sc1, sc0) and np.array_equal(u1, u0)
    assert np.array_equal(h1, h0)
    D = O.gram(w.base, w.Xd, gamma=w.gamma)
    T = None if w.Xt is None else O.gram(w.base, w.Xt, gamma=w.gamma)
    solve = O.minres if solver == 1 else O.cg
    ao, _, _, _ = solve(O.kernel_terms(kernel), D, T, w.train_first, w.train_second, w.y, w.lam, 20)
    assert rel(a1, ao) <= 1e-4


def test_nccl_world1_early_stopping(pair):
    """The early-stopping fit gathers its validation labels and scores with NCCL (grouped
    broadcasts each iteration) and equals the single-GPU result."""
    nc, plain = pair
    w, vlab = synth.parity_grid("chessboard", 12, 12, seed=0)
    D = dev(np.ascontiguousarray(O.gram(O.BASE_LINEAR, w.Xd), dtype=np.float32))
    T = dev(np.ascontiguousarray(O.gram(O.BASE_LINEAR, w.Xt), dtype=np.float32))
    res = []
    for c in (nc, plain):
        c.set_option(G.OPT_SOLVER, G.SOLVER_MINRES)
        c.reset_stats()
        a, best, auc, iters, hist = c.fit_early_stopping(
            D, T, dev(w.train_first), dev(w.train_second), dev(w.y), dev(w.test_first), dev(w.test_second), dev(vlab),
            G.gvt_kernel_terms(G.KRONECKER), 1e-5, 10, w.n)
        res.append((a.cpu().numpy(), best, auc, iters, hist, _collectives(c)))
        c.set_option(G.OPT_SOLVER, G.SOLVER_CG)
    assert res[0][5] > 0 and res[1][5] == 0
    assert np.array_equal(res[0][0], res[1][0]) and res[0][1:4] == res[1][1:4]
    ob, oauc, oit, _, _ = O.fit_early_stopping(O.kernel_terms(O.KRONECKER), O.gram(O.BASE_LINEAR, w.Xd),
                                               O.gram(O.BASE_LINEAR, w.Xt), w.train_first, w.train_second, w.y,
                                               w.test_first, w.test_second, vlab, 1e-5, 10, w.n, "minres")
    assert (res[0][1], res[0][3]) == (ob, oit)


def test_nccl_world1_stats_and_reinit(pair):
    """gvt_get_stats reports world 1 with the communicator; re-initialising replaces it; world 1
    without an id returns to single-GPU mode (no collectives)."""
    nc, _ = pair
    assert nc.stats()["world"] == 1
    c = G.Context(0)
    try:
        c.comm_init(G.gvt_nccl_unique_id(), 0, 1)
        c.comm_init(G.gvt_nccl_unique_id(), 0, 1)   # replaces the first communicator
        w = synth.config1()
        D = c.gram(w.base, dev(w.Xd), gamma=w.gamma)
        T = c.gram(w.base, dev(w.Xt), gamma=w.gamma)
        terms = G.gvt_kernel_terms(G.KRONECKER)
        c.reset_stats()
        c.matvec(D, T, dev(w.train_first), dev(w.train_second), dev(w.train_first), dev(w.train_second),
                 dev(w.y), terms)
        assert _collectives(c) > 0
        with pytest.raises(G.GvtError) as e:
            c.comm_init(b"\0" * 128, 1, 1)          # rank outside [0, world)
        assert e.value.code == G.E_PARAM
    finally:
        c.close()
