"""Used-object compaction of fits (GVT_OPT_COMPACT = 2 forces it on these small tables; PAPER.md
Table 1's unique counts m, q):
a training sample over a subset of a larger object table is solved on the sub-Grams of the used
objects.  GPU vs the fp64 oracle (CG weights, relative L2 <= 1e-4), on vs off, early stopping,
and a NaN-poisoned Gram proving the unused objects are never read (-m gpu)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O
import synth

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2009_01054_b200 as G

K_ALL = [G.LINEAR, G.POLY2D, G.GAUSSIAN, G.KRONECKER, G.SYMMETRIC, G.ANTISYMMETRIC, G.RANKING, G.MLPK,
         G.CARTESIAN]


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def rel(x, ref):
    return float(np.linalg.norm(np.asarray(x, np.float64) - ref) / np.linalg.norm(ref))


@pytest.fixture(scope="module")
def ctx():
    c = G.Context(0)
    yield c
    c.close()


def subset_problem(kernel, seed, m=300, q=200, used_m=50, used_q=40, n=700):
    """Pairs over a random subset of a larger object table (ids scattered, not contiguous)."""
    rng = np.random.default_rng(seed)
    hom = kernel in G.HOMOGENEOUS_KERNELS
    q = m if hom else q
    Xd = rng.standard_normal((m, 12)).astype(np.float32)
    Xt = None if hom else rng.standard_normal((q, 12)).astype(np.float32)
    D = O.gram(O.BASE_GAUSSIAN, Xd, gamma=1 / 12).astype(np.float32)
    T = None if hom else O.gram(O.BASE_GAUSSIAN, Xt, gamma=1 / 12).astype(np.float32)
    ud = rng.choice(m, used_m, replace=False)
    ut = ud if hom else rng.choice(q, used_q, replace=False)
    f = ud[rng.integers(0, len(ud), n)].astype(np.int32)
    s = ut[rng.integers(0, len(ut), n)].astype(np.int32)
    y = rng.standard_normal(n).astype(np.float32)
    return D, T, f, s, y


@pytest.mark.parametrize("engine", [G.ENGINE_SPARSE, G.ENGINE_DENSE], ids=["sparse", "dense"])
@pytest.mark.parametrize("kernel", K_ALL)
def test_compacted_fit_matches_oracle(ctx, kernel, engine):
    D, T, f, s, y = subset_problem(kernel, 100 + kernel)
    terms = G.gvt_kernel_terms(kernel)
    ao, _, _, _ = O.cg(O.kernel_terms(kernel), D.astype(np.float64), None if T is None else T.astype(np.float64),
                       f, s, y, 1.0, 30)
    ctx.set_option(G.OPT_ENGINE, engine)
    try:
        res = {}
        for compact in (2, 0):
            ctx.set_option(G.OPT_COMPACT, compact)
            a, it, _, code = ctx.fit(dev(D), None if T is None else dev(T), dev(f), dev(s), dev(y), terms, 1.0, 30)
            assert code == G.OK and it == 30
            res[compact] = rel(a.cpu().numpy(), ao)
        # the C1 weight gate (1e-4, reading S30) where the system is well conditioned; on the
        # ill-conditioned ones (Poly2D's (D + T)^2 values) fp32 CG drifts either way, and the
        # compacted fit must be no worse than the full-Gram fit
        assert res[2] <= max(1e-4, 3.0 * res[0]), res
    finally:
        ctx.set_option(G.OPT_COMPACT, 1)
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)


@pytest.mark.parametrize("kernel", [G.KRONECKER, G.SYMMETRIC, G.MLPK])
def test_unused_objects_are_never_read(ctx, kernel):
    """Grams with NaN in every row and column of an unused object: the compacted fits (dense and
    sparse engines) are finite and at oracle parity; without compaction the NaNs reach the result."""
    D, T, f, s, y = subset_problem(kernel, 200 + kernel)
    terms = G.gvt_kernel_terms(kernel)
    ao, _, _, _ = O.cg(O.kernel_terms(kernel), D.astype(np.float64), None if T is None else T.astype(np.float64),
                       f, s, y, 1.0, 20)

    def poison(M, used):
        P = M.copy()
        unused = np.setdiff1d(np.arange(M.shape[0]), used)
        P[unused, :] = np.nan
        P[:, unused] = np.nan
        return P

    hom = T is None
    Dp = poison(D, np.union1d(f, s) if hom else np.unique(f))
    Tp = None if hom else poison(T, np.unique(s))
    ctx.set_option(G.OPT_ENGINE, G.ENGINE_DENSE)
    try:
        ctx.set_option(G.OPT_COMPACT, 0)  # reference error: the full-Gram fit on the clean Grams
        e0 = rel(ctx.fit(dev(D), None if hom else dev(T), dev(f), dev(s), dev(y), terms, 1.0, 20)[0].cpu().numpy(), ao)
        ctx.set_option(G.OPT_COMPACT, 2)
        a, _, _, _ = ctx.fit(dev(Dp), None if hom else dev(Tp), dev(f), dev(s), dev(y), terms, 1.0, 20)
        a = a.cpu().numpy()
        assert np.all(np.isfinite(a)) and rel(a, ao) <= max(1e-4, 3.0 * e0), (rel(a, ao), e0)
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_SPARSE)
        a1, _, _, _ = ctx.fit(dev(Dp), None if hom else dev(Tp), dev(f), dev(s), dev(y), terms, 1.0, 20)
        assert np.all(np.isfinite(a1.cpu().numpy()))
        # the test can see a full-Gram read: the uncompacted sparse stage 2 dots whole Gram rows
        # (NaN x 0 = NaN at the unused columns), so p.Ap is NaN and CG reports a breakdown
        ctx.set_option(G.OPT_COMPACT, 0)
        a0, _, _, code0 = ctx.fit(dev(Dp), None if hom else dev(Tp), dev(f), dev(s), dev(y), terms, 1.0, 20,
                                  raise_on_breakdown=False)
        assert code0 == G.E_BREAKDOWN or not np.all(np.isfinite(a0.cpu().numpy()))
    finally:
        ctx.set_option(G.OPT_COMPACT, 1)
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)


def test_compacted_early_stopping_equals_plain_fit(ctx):
    """Early stopping on a subset whose validation pairs use the training objects: both runs are
    compacted the same way, so a_best is bit-identical to a plain fit of best_iter iterations."""
    D, T, f, s, y = subset_problem(G.SYMMETRIC, 7, n=900)
    rng = np.random.default_rng(8)
    objs = np.union1d(f, s)
    vf = objs[rng.integers(0, len(objs), 300)].astype(np.int32)
    vs = objs[rng.integers(0, len(objs), 300)].astype(np.int32)
    vlab = (rng.standard_normal(300) > 0).astype(np.float32)
    terms = G.gvt_kernel_terms(G.SYMMETRIC)
    ctx.set_option(G.OPT_SOLVER, G.SOLVER_MINRES)
    ctx.set_option(G.OPT_COMPACT, 2)  # (the table is below the auto threshold)
    try:
        a, best, best_auc, it_run, hist = ctx.fit_early_stopping(dev(D), None, dev(f), dev(s), dev(y), dev(vf),
                                                                 dev(vs), dev(vlab), terms, 1.0, 13, 12)
        ap, _, _, _ = ctx.fit(dev(D), None, dev(f), dev(s), dev(y), terms, 1.0, best)
        assert torch.equal(a, ap)
        # and the compacted result equals the uncompacted one to fp32 rounding
        ctx.set_option(G.OPT_COMPACT, 0)
        a0, best0, _, _, _ = ctx.fit_early_stopping(dev(D), None, dev(f), dev(s), dev(y), dev(vf), dev(vs),
                                                    dev(vlab), terms, 1.0, 13, 12)
        assert best0 == best and rel(a.cpu().numpy(), a0.cpu().numpy().astype(np.float64)) <= 1e-4
    finally:
        ctx.set_option(G.OPT_COMPACT, 1)
        ctx.set_option(G.OPT_SOLVER, G.SOLVER_CG)


@pytest.mark.parametrize("engine", [G.ENGINE_SPARSE, G.ENGINE_DENSE], ids=["sparse", "dense"])
@pytest.mark.parametrize("kernel", K_ALL)
def test_compacted_matvec_and_predict_match_oracle(ctx, kernel, engine):
    """gvt_matvec / pairwise_predict with in- and out-samples over subsets of the object table run
    on the cross-Grams of the used objects (rectangular path, variant by cost); Cartesian keeps the
    square path.  Against the oracle's per-term GVT at the matvec tolerance (1e-5), and with a
    NaN-poisoned table outside the used objects for the compacted kernels."""
    D, T, f, s, _ = subset_problem(kernel, 300 + kernel)
    rng = np.random.default_rng(400 + kernel)
    hom = T is None
    # test pairs over a different subset of objects than the training pairs
    m = D.shape[0]
    q = m if hom else T.shape[0]
    od = rng.choice(m, 30, replace=False)
    ot = od if hom else rng.choice(q, 25, replace=False)
    tf = od[rng.integers(0, len(od), 500)].astype(np.int32)
    ts = ot[rng.integers(0, len(ot), 500)].astype(np.int32)
    a = synth.random_vector(kernel, len(f))
    terms = G.gvt_kernel_terms(kernel)
    ref = O.gvt_matvec(O.kernel_terms(kernel), D.astype(np.float64), None if hom else T.astype(np.float64), tf, ts,
                       f, s, a)
    ctx.set_option(G.OPT_ENGINE, engine)
    try:
        for compact in (2, 0):
            ctx.set_option(G.OPT_COMPACT, compact)
            u = ctx.predict(dev(D), None if hom else dev(T), dev(tf), dev(ts), dev(f), dev(s), dev(a), terms)
            assert rel(u.cpu().numpy(), ref) <= 1e-5, (compact, rel(u.cpu().numpy(), ref))
        if kernel != G.CARTESIAN:
            used_d = np.union1d(np.union1d(f, s), np.union1d(tf, ts)) if hom else np.union1d(f, tf)
            Dp = D.copy()
            bad = np.setdiff1d(np.arange(m), used_d)
            Dp[bad, :] = np.nan
            Dp[:, bad] = np.nan
            Tp = None
            if not hom:
                Tp = T.copy()
                badt = np.setdiff1d(np.arange(q), np.union1d(s, ts))
                Tp[badt, :] = np.nan
                Tp[:, badt] = np.nan
            ctx.set_option(G.OPT_COMPACT, 2)
            u = ctx.predict(dev(Dp), None if hom else dev(Tp), dev(tf), dev(ts), dev(f), dev(s), dev(a), terms)
            u = u.cpu().numpy()
            assert np.all(np.isfinite(u)) and rel(u, ref) <= 1e-5
    finally:
        ctx.set_option(G.OPT_COMPACT, 1)
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)


@pytest.mark.parametrize("exchange", [0, 1], ids=["S-allgather", "u-reduce"])
@pytest.mark.parametrize("kernel", [G.KRONECKER, G.MLPK, G.POLY2D])
def test_compaction_with_emulated_slabs(ctx, kernel, exchange):
    """Compaction composes with the data-parallel slab decomposition (3 emulated slabs, both
    exchanges): the slabs are cut over the compacted object numbering."""
    D, T, f, s, y = subset_problem(kernel, 500 + kernel)
    terms = G.gvt_kernel_terms(kernel)
    ao, _, _, _ = O.cg(O.kernel_terms(kernel), D.astype(np.float64), None if T is None else T.astype(np.float64),
                       f, s, y, 1.0, 25)
    ctx.set_option(G.OPT_COMPACT, 0)
    e0 = rel(ctx.fit(dev(D), None if T is None else dev(T), dev(f), dev(s), dev(y), terms, 1.0, 25)[0].cpu().numpy(),
             ao)
    ctx.set_option(G.OPT_COMPACT, 2)
    ctx.set_option(G.OPT_SLABS, 3)
    ctx.set_option(G.OPT_EXCHANGE, exchange)
    try:
        a, it, _, _ = ctx.fit(dev(D), None if T is None else dev(T), dev(f), dev(s), dev(y), terms, 1.0, 25)
        assert it == 25 and rel(a.cpu().numpy(), ao) <= max(1e-4, 3.0 * e0)
    finally:
        ctx.set_option(G.OPT_SLABS, 1)
        ctx.set_option(G.OPT_EXCHANGE, 0)
        ctx.set_option(G.OPT_COMPACT, 1)
