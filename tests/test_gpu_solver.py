"""GPU parity of the paper's solver and early-stopping protocol (-m gpu), through the C ABI:
MINRES, validation AUC and the early-stopping rule,
against the fp64 oracle (O5b, O8, oracle.fit_early_stopping) on the same seeded inputs.
Tolerances: the north star's (weights after a fixed iteration count <= 1e-4 relative L2 on
C1, predictions max-abs <= 1e-4); the AUC is exact given the scores (integer counting on both
sides over the same fp32 scores)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O
import synth

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2009_01054_b200 as G

HOM = G.HOMOGENEOUS_KERNELS


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def rel(x, ref):
    x, ref = np.asarray(x, np.float64), np.asarray(ref, np.float64)
    nr = np.linalg.norm(ref)
    return np.linalg.norm(x - ref) / (nr if nr > 1e-30 else 1.0)


def f32(x):
    return None if x is None else np.ascontiguousarray(x, dtype=np.float32)


@pytest.fixture(scope="module")
def ctx():
    c = G.Context(0)
    yield c
    c.close()


@pytest.fixture
def minres_ctx(ctx):
    ctx.set_option(G.OPT_SOLVER, G.SOLVER_MINRES)
    yield ctx
    ctx.set_option(G.OPT_SOLVER, G.SOLVER_CG)
    ctx.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)


# ----------------------------------------------------------------------------- AUC
def test_auc_exact_against_oracle_definition(ctx):
    """gvt_auc (radix sort + integer counting) equals the oracle's brute-force Mann-Whitney
    definition on the same fp32 scores exactly, with heavy ties, 0/1 and -1/+1 labels, sizes
    from 2 to 30 000 (several sort tiles, ragged)."""
    rng = np.random.default_rng(11)
    for n in (2, 3, 17, 1000, 4097, 30_000):
        lab = rng.integers(0, 2, n).astype(np.float32)
        lab[0], lab[-1] = 0, 1
        for ties in (False, True):
            sc = rng.standard_normal(n).astype(np.float32)
            if ties:
                sc = np.round(sc * 4) / 4
            a = ctx.auc(dev(lab), dev(sc))
            assert a == O.auc(lab, sc.astype(np.float64)), (n, ties)
            assert ctx.auc(dev(2 * lab - 1), dev(sc)) == a
    # host buffers go through the same path
    assert ctx.auc(lab, sc) == O.auc(lab, sc.astype(np.float64))
    with pytest.raises(G.GvtError) as e:
        ctx.auc(dev(np.ones(5, np.float32)), dev(np.arange(5, dtype=np.float32)))
    assert e.value.code == G.E_PARAM


# ----------------------------------------------------------------------------- MINRES
def test_minres_scalar_systems(minres_ctx):
    """2I -> y / 2 in one iteration; y = 0 -> a = 0 after 0 iterations (SPEC minres_solve)."""
    f = np.repeat(np.arange(3), 2).astype(np.int32)
    s = np.tile(np.arange(2), 3).astype(np.int32)
    y = np.array([1.0, -2.0, 0.5, 4.0, 3.0, -1.0], np.float32)
    kron = G.gvt_kernel_terms(G.KRONECKER)
    I3, I2 = dev(np.eye(3, dtype=np.float32)), dev(np.eye(2, dtype=np.float32))
    a, it, hist, code = minres_ctx.fit(I3, I2, dev(f), dev(s), dev(y), kron, 1.0, 5)
    assert code == G.OK and it == 1
    assert np.allclose(a.cpu().numpy(), y / 2, atol=1e-7)
    a, it, hist, code = minres_ctx.fit(I3, I2, dev(f), dev(s), dev(np.zeros(6, np.float32)), kron, 1.0, 5)
    assert it == 0 and np.all(a.cpu().numpy() == 0)


@pytest.mark.parametrize("engine", [G.ENGINE_SPARSE, G.ENGINE_DENSE])
def test_minres_c1_weights_predictions_and_monotone_residual(minres_ctx, engine):
    """C1: 50 MINRES iterations on the GPU vs the oracle's fp64 MINRES: weights <= 1e-4
    relative L2, predictions max-abs <= 1e-4, and the residual history is non-increasing."""
    minres_ctx.set_option(G.OPT_ENGINE, engine)
    w = synth.config1()
    kron = G.gvt_kernel_terms(G.KRONECKER)
    D = O.gram(w.base, w.Xd, gamma=w.gamma)
    T = O.gram(w.base, w.Xt, gamma=w.gamma)
    Dg, Tg = dev(f32(D)), dev(f32(T))
    a, it, hist, code = minres_ctx.fit(Dg, Tg, dev(w.train_first), dev(w.train_second), dev(w.y), kron, w.lam,
                                       w.iters)
    assert code == G.OK and it == w.iters
    assert all(hist[k + 1] <= hist[k] for k in range(len(hist) - 1))
    ao, it_o, hist_o, _ = O.minres(O.kernel_terms(O.KRONECKER), D, T, w.train_first, w.train_second, w.y, w.lam,
                                   w.iters)
    assert rel(a.cpu().numpy(), ao) <= 1e-4
    assert hist[-1] <= 1e-5
    scores = minres_ctx.predict(Dg, Tg, dev(w.test_first), dev(w.test_second), dev(w.train_first),
                                dev(w.train_second), a, kron).cpu().numpy()
    ref = O.gvt_matvec(O.kernel_terms(O.KRONECKER), D, T, w.test_first, w.test_second, w.train_first,
                       w.train_second, ao)
    assert np.abs(scores - ref).max() <= 1e-4


@pytest.mark.parametrize("kernel", [G.KRONECKER, G.SYMMETRIC, G.ANTISYMMETRIC, G.MLPK, G.POLY2D, G.RANKING,
                                    G.CARTESIAN, G.LINEAR])
def test_minres_early_iterates_all_kernels(minres_ctx, kernel):
    """Every kernel's operator inside MINRES: after 6 iterations on a seeded 300-pair instance the
    GPU iterate equals the oracle's within 1e-4 (early iterates, before Lanczos rounding grows)
    and the residual histories agree within 1e-4."""
    hom = kernel in HOM
    w = synth.tiny(21, m=30, q=25, n=300, n_out=10, homogeneous=hom, duplicates=False)
    D = O.gram(G.BASE_GAUSSIAN, w.Xd, gamma=0.5)
    T = None if hom else O.gram(G.BASE_GAUSSIAN, w.Xt, gamma=0.5)
    terms = G.gvt_kernel_terms(kernel)
    a, it, hist, code = minres_ctx.fit(dev(f32(D)), None if hom else dev(f32(T)), dev(w.train_first),
                                       dev(w.train_second), dev(w.y), terms, 0.5, 6)
    ao, it_o, hist_o, _ = O.minres(O.kernel_terms(kernel), f32(D), f32(T), w.train_first, w.train_second, w.y, 0.5, 6)
    assert it == it_o
    assert rel(a.cpu().numpy(), ao) <= 1e-4
    assert np.allclose(hist, hist_o, rtol=1e-4, atol=1e-7)


def test_minres_residual_mode_stops(minres_ctx):
    """rel_tol > 0: MINRES stops at the first iteration with ||r_k|| / ||y|| <= rel_tol (the
    oracle stops at the same iteration on C1).  The fp32 Lanczos vectors lose orthogonality
    sooner than the oracle's fp64 ones (measured on C1: histories equal to 4 digits for k <= 8,
    then the GPU stagnates at k = 9-10, the oracle at k = 15-16), so tol = 0.08 sits between the
    iteration-4 and -5 residuals 0.116 / 0.059, inside the lockstep range."""
    w = synth.config1()
    D = O.gram(w.base, w.Xd, gamma=w.gamma)
    T = O.gram(w.base, w.Xt, gamma=w.gamma)
    kron = G.gvt_kernel_terms(G.KRONECKER)
    a, it, hist, code = minres_ctx.fit(dev(f32(D)), dev(f32(T)), dev(w.train_first), dev(w.train_second), dev(w.y),
                                       kron, w.lam, 200, 0.08)
    _, it_o, _, _ = O.minres(O.kernel_terms(O.KRONECKER), D, T, w.train_first, w.train_second, w.y, w.lam, 200, 0.08)
    assert it == it_o == 5 and hist[-1] <= 0.08 < hist[-2]


# ----------------------------------------------------------------------------- early stopping
@pytest.mark.parametrize("solver", [G.SOLVER_MINRES, G.SOLVER_CG])
@pytest.mark.parametrize("engine", [G.ENGINE_SPARSE, G.ENGINE_DENSE])
def test_early_stopping_chessboard(ctx, solver, engine):
    """SPEC.md's chessboard 12x12 case (Kronecker, lambda = 1e-5, patience 10): same best
    iteration, AUC history and stopping iteration as the oracle's fit_early_stopping; the
    device rule agrees with the rule applied to the device's own AUC history; a_best scored
    directly gives the best AUC."""
    ctx.set_option(G.OPT_SOLVER, solver)
    ctx.set_option(G.OPT_ENGINE, engine)
    try:
        w, vlab = synth.parity_grid("chessboard", 12, 12, seed=0)
        D = O.gram(O.BASE_LINEAR, w.Xd)
        T = O.gram(O.BASE_LINEAR, w.Xt)
        kron = G.gvt_kernel_terms(G.KRONECKER)
        Dg, Tg = dev(f32(D)), dev(f32(T))
        a, best, best_auc, iters, hist = ctx.fit_early_stopping(
            Dg, Tg, dev(w.train_first), dev(w.train_second), dev(w.y), dev(w.test_first), dev(w.test_second),
            dev(vlab), kron, 1e-5, 10, w.n)
        ob, oauc, oit, ohist, oa = O.fit_early_stopping(O.kernel_terms(O.KRONECKER), D, T, w.train_first,
                                                        w.train_second, w.y, w.test_first, w.test_second, vlab,
                                                        1e-5, 10, w.n, "minres" if solver else "cg")
        assert (best, iters) == (ob, oit)
        assert best_auc == pytest.approx(oauc, abs=1e-6)
        assert np.allclose(hist, ohist, atol=1e-6)
        rb, rauc, rit, _ = O.early_stop_rule(list(hist), 10)
        assert (rb, rauc, rit) == (best, best_auc, iters)
        sc = ctx.predict(Dg, Tg, dev(w.test_first), dev(w.test_second), dev(w.train_first), dev(w.train_second), a,
                         kron)
        assert ctx.auc(dev(vlab), sc) == pytest.approx(best_auc, abs=1e-6)
    finally:
        ctx.set_option(G.OPT_SOLVER, G.SOLVER_CG)
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)


@pytest.mark.parametrize("solver", [G.SOLVER_MINRES, G.SOLVER_CG])
@pytest.mark.parametrize("kernel", [G.KRONECKER, G.SYMMETRIC, G.MLPK])
def test_early_stopping_weights_equal_plain_fit(ctx, solver, kernel):
    """The [inner; validation] out sample does not perturb the solve: with patience large enough
    to run to max_iter, a_best is bit-identical to a plain fit of best_iter iterations, and the
    AUC of its direct validation scores matches the recorded best within 1e-4.  Seeded
    C3-shaped instance (homogeneous kernels) or C1 (Kronecker); labels y > 0 as the classes."""
    ctx.set_option(G.OPT_SOLVER, solver)
    ctx.set_option(G.OPT_ENGINE, G.ENGINE_DENSE)  # the same engine for both fits (not the single-CTA solver)
    try:
        if kernel == G.KRONECKER:
            w = synth.config1()
            vf, vs = w.test_first, w.test_second
        else:
            w = synth.config3(n=20_000, n_test=5_000)
            vf, vs = w.test_first, w.test_second
        D = O.gram(w.base, w.Xd, gamma=w.gamma)
        T = None if w.Xt is None else O.gram(w.base, w.Xt, gamma=w.gamma)
        Dg, Tg = dev(f32(D)), (None if T is None else dev(f32(T)))
        terms = G.gvt_kernel_terms(kernel)
        rng = np.random.default_rng(3)
        vlab = (rng.standard_normal(len(vf)) > 0).astype(np.float32)
        iters = 12
        a, best, best_auc, it_run, hist = ctx.fit_early_stopping(
            Dg, Tg, dev(w.train_first), dev(w.train_second), dev(w.y), dev(vf), dev(vs), dev(vlab), terms, w.lam,
            iters + 1, iters)
        assert it_run == iters and 1 <= best <= iters
        ap, itp, _, _ = ctx.fit(Dg, Tg, dev(w.train_first), dev(w.train_second), dev(w.y), terms, w.lam, best)
        assert torch.equal(a, ap)
        sc = ctx.predict(Dg, Tg, dev(vf), dev(vs), dev(w.train_first), dev(w.train_second), a, terms)
        assert ctx.auc(dev(vlab), sc) == pytest.approx(best_auc, abs=1e-4)
        assert best_auc == np.max(hist) and hist[best - 1] == best_auc
    finally:
        ctx.set_option(G.OPT_SOLVER, G.SOLVER_CG)
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)


def test_early_stopping_errors(ctx):
    w, vlab = synth.parity_grid("tablecloth", 6, 6, seed=1)
    kron = G.gvt_kernel_terms(G.KRONECKER)
    D = dev(f32(O.gram(O.BASE_LINEAR, w.Xd)))
    T = dev(f32(O.gram(O.BASE_LINEAR, w.Xt)))
    args = (D, T, dev(w.train_first), dev(w.train_second), dev(w.y), dev(w.test_first), dev(w.test_second))
    with pytest.raises(G.GvtError) as e:
        ctx.fit_early_stopping(*args, dev(np.ones_like(vlab)), kron, 1e-3, 3, 20)
    assert e.value.code == G.E_PARAM
    with pytest.raises(G.GvtError) as e:
        ctx.fit_early_stopping(*args, dev(vlab), kron, 1e-3, 0, 20)
    assert e.value.code == G.E_PARAM


# ----------------------------------------------------------------------------- single-reduction CG
@pytest.fixture
def cgg_ctx(ctx):
    ctx.set_option(G.OPT_CG_VARIANT, 1)
    yield ctx
    ctx.set_option(G.OPT_CG_VARIANT, 0)
    ctx.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)


@pytest.mark.parametrize("engine", [G.ENGINE_SPARSE, G.ENGINE_DENSE])
def test_chronopoulos_gear_cg_matches_oracle_cg(cgg_ctx, engine):
    """GVT_OPT_CG_VARIANT = 1 has the Hestenes-Stiefel iterates in exact arithmetic: on C1 its 50
    iterations match the oracle's CG weights (<= 1e-4) and residual history, and residual mode
    stops at the oracle's iteration; per iteration it launches 3 solver kernels instead of the separate
    Hestenes-Stiefel kernels' 5 (on the dense engine Hestenes-Stiefel CG runs the fused tail, one launch)."""
    cgg_ctx.set_option(G.OPT_ENGINE, engine)
    w = synth.config1()
    D = O.gram(w.base, w.Xd, gamma=w.gamma)
    T = O.gram(w.base, w.Xt, gamma=w.gamma)
    Dg, Tg = dev(f32(D)), dev(f32(T))
    kron = G.gvt_kernel_terms(G.KRONECKER)
    args = (Dg, Tg, dev(w.train_first), dev(w.train_second), dev(w.y), kron, w.lam)
    a, it, hist, code = cgg_ctx.fit(*args, w.iters)
    ao, _, hist_o, _ = O.cg(O.kernel_terms(O.KRONECKER), D, T, w.train_first, w.train_second, w.y, w.lam, w.iters)
    assert code == G.OK and it == w.iters
    assert rel(a.cpu().numpy(), ao) <= 1e-4
    # fp32 recurrences drift from the fp64 ones once the Krylov vectors lose orthogonality
    # (on C1 the histories agree to 5 digits for k <= 7 and drift from k = 8, as for MINRES, reading M3)
    assert np.allclose(hist[:8], hist_o[:8], rtol=1e-4, atol=1e-7)
    a2, it2, h2, _ = cgg_ctx.fit(*args, 200, rel_tol=0.05)
    _, it2o, _, _ = O.cg(O.kernel_terms(O.KRONECKER), D, T, w.train_first, w.train_second, w.y, w.lam, 200,
                         rel_tol=0.05)
    assert it2 == it2o == 6 and h2[-1] <= 0.05 < h2[-2]
    # launch accounting (eager, profiled): solver kernels per iteration
    cgg_ctx.set_option(G.OPT_PROFILE, 1)
    per = {}
    for variant in (0, 1):
        cgg_ctx.set_option(G.OPT_CG_VARIANT, variant)
        cgg_ctx.reset_stats()
        cgg_ctx.fit(*args, 10)
        k = cgg_ctx.stats()["kinds"]
        per[variant] = k["cg_vector"]["count"] + k["cg_scalar"]["count"]
    cgg_ctx.set_option(G.OPT_PROFILE, 0)
    if engine == G.ENGINE_DENSE:  # the dense engine's Hestenes-Stiefel CG runs the fused tail: 1 launch / iteration
        assert per[0] < per[1]
    else:
        assert per[1] < per[0]


@pytest.mark.parametrize("kernel", [G.SYMMETRIC, G.MLPK, G.POLY2D, G.CARTESIAN])
@pytest.mark.parametrize("n", [1, 5, 1185, 30011])
def test_chronopoulos_gear_cg_kernels_and_ragged(cgg_ctx, kernel, n):
    hom = kernel in HOM
    rng = np.random.default_rng(n + kernel)
    m, q = 37, 29
    D32 = f32(O.gram(G.BASE_GAUSSIAN, rng.standard_normal((m, 4)), gamma=0.25))
    T32 = None if hom else f32(O.gram(G.BASE_GAUSSIAN, rng.standard_normal((q, 4)), gamma=0.25))
    f = rng.integers(0, m, n).astype(np.int32)
    s = rng.integers(0, m if hom else q, n).astype(np.int32)
    y = rng.standard_normal(n).astype(np.float32)
    terms = G.gvt_kernel_terms(kernel)
    a, it, _, _ = cgg_ctx.fit(dev(D32), None if hom else dev(T32), dev(f), dev(s), dev(y), terms, 1.0, 8)
    ao, ito, _, _ = O.cg(O.kernel_terms(kernel), D32, T32, f, s, y, 1.0, 8)
    # an n <= 8 system converges exactly within n steps in fp64 (the oracle stops at r = 0); the fp32
    # residual is rounding noise there, so only the weights are compared in that case
    assert it == ito or n <= 8
    # the single-reduction form is within 1e-4 of the oracle, or no worse than 3x the fp32
    # Hestenes-Stiefel CG on the same instance (duplicate symmetric pairs make these systems
    # ill-conditioned; measured 1.3e-4 at n = 1185, Symmetric)
    cgg_ctx.set_option(G.OPT_CG_VARIANT, 0)
    ah, _, _, _ = cgg_ctx.fit(dev(D32), None if hom else dev(T32), dev(f), dev(s), dev(y), terms, 1.0, 8)
    cgg_ctx.set_option(G.OPT_CG_VARIANT, 1)
    assert rel(a.cpu().numpy(), ao) <= max(1e-4, 3 * rel(ah.cpu().numpy(), ao))


@pytest.mark.parametrize("solver,variant", [(0, 0), (0, 1), (1, 0)], ids=["cg", "cg-cgg", "minres"])
def test_long_fixed_iteration_fit_stays_finite(ctx, solver, variant):
    """Reading S32: far more iterations than convergence needs (C1, 300) end as converged at the
    residual floor instead of underflowing into 0/0; the weights equal the oracle's converged
    solution."""
    ctx.set_option(G.OPT_SOLVER, solver)
    ctx.set_option(G.OPT_CG_VARIANT, variant)
    try:
        w = synth.config1()
        D = O.gram(w.base, w.Xd, gamma=w.gamma)
        T = O.gram(w.base, w.Xt, gamma=w.gamma)
        kron = G.gvt_kernel_terms(G.KRONECKER)
        a, it, hist, code = ctx.fit(dev(f32(D)), dev(f32(T)), dev(w.train_first), dev(w.train_second), dev(w.y),
                                    kron, w.lam, 300)
        assert code == G.OK and it <= 300 and np.all(np.isfinite(a.cpu().numpy()))
        ao, _, _, _ = O.cg(O.kernel_terms(O.KRONECKER), D, T, w.train_first, w.train_second, w.y, w.lam, 60)
        assert rel(a.cpu().numpy(), ao) <= 1e-4
    finally:
        ctx.set_option(G.OPT_SOLVER, 0)
        ctx.set_option(G.OPT_CG_VARIANT, 0)


# ----------------------------------------------------------------------------- single-CTA whole-fit solver
def test_tiny_engine_c1_matches_oracle(ctx):
    """GVT_OPT_ENGINE = 3: the whole C1 CG fit in one single-CTA launch; weights (<= 1e-4),
    predictions (<= 1e-4 max-abs), residual-mode stop and the residual history match the oracle;
    auto selects it on C1; an ineligible problem is an error, not a silent fallback."""
    w = synth.config1()
    D = O.gram(w.base, w.Xd, gamma=w.gamma)
    T = O.gram(w.base, w.Xt, gamma=w.gamma)
    Dg, Tg = dev(f32(D)), dev(f32(T))
    kron = G.gvt_kernel_terms(G.KRONECKER)
    args = (Dg, Tg, dev(w.train_first), dev(w.train_second), dev(w.y), kron, w.lam)
    ao, _, hist_o, _ = O.cg(O.kernel_terms(O.KRONECKER), D, T, w.train_first, w.train_second, w.y, w.lam, w.iters)
    try:
        for engine in (G.ENGINE_TINY, G.ENGINE_AUTO):
            ctx.set_option(G.OPT_ENGINE, engine)
            ctx.reset_stats()
            a, it, hist, code = ctx.fit(*args, w.iters)
            st = ctx.stats()
            assert st["last_engine"] == 3 and st["kinds"]["tiny_cg"]["count"] == 1
            assert code == G.OK and it == w.iters
            assert rel(a.cpu().numpy(), ao) <= 1e-4
            assert np.allclose(hist[:8], hist_o[:8], rtol=1e-4, atol=1e-7)
        sc = ctx.predict(Dg, Tg, dev(w.test_first), dev(w.test_second), dev(w.train_first), dev(w.train_second), a,
                         kron).cpu().numpy()
        ref = O.gvt_matvec(O.kernel_terms(O.KRONECKER), D, T, w.test_first, w.test_second, w.train_first,
                           w.train_second, ao)
        assert np.abs(sc - ref).max() <= 1e-4
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_TINY)
        a2, it2, h2, _ = ctx.fit(*args, 200, rel_tol=0.05)
        _, it2o, _, _ = O.cg(O.kernel_terms(O.KRONECKER), D, T, w.train_first, w.train_second, w.y, w.lam, 200,
                             rel_tol=0.05)
        assert it2 == it2o and h2[-1] <= 0.05 < h2[-2]
        with pytest.raises(G.GvtError) as e:  # Symmetric is not eligible for the single-CTA solver
            ctx.fit(Dg, None, dev(w.train_first % 40), dev(w.train_second % 40), dev(w.y),
                    G.gvt_kernel_terms(G.SYMMETRIC), 1.0, 5)
        assert e.value.code == G.E_PARAM
    finally:
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)


@pytest.mark.parametrize("m,q,n", [(1, 1, 1), (3, 2, 5), (17, 29, 300), (64, 100, 4000), (60, 100, 9000)])
def test_tiny_engine_shapes(ctx, m, q, n):
    """Ragged shapes through the single-CTA solver (duplicates, n not a multiple of the block size,
    n larger than the thread count) against the oracle's CG on the same fp32 inputs."""
    rng = np.random.default_rng(m * 1000 + n)
    D32 = f32(O.gram(G.BASE_GAUSSIAN, rng.standard_normal((m, 4)), gamma=0.25))
    T32 = f32(O.gram(G.BASE_GAUSSIAN, rng.standard_normal((q, 4)), gamma=0.25))
    f = rng.integers(0, m, n).astype(np.int32)
    s = rng.integers(0, q, n).astype(np.int32)
    y = rng.standard_normal(n).astype(np.float32)
    kron = G.gvt_kernel_terms(G.KRONECKER)
    ctx.set_option(G.OPT_ENGINE, G.ENGINE_TINY)
    try:
        a, it, _, _ = ctx.fit(dev(D32), dev(T32), dev(f), dev(s), dev(y), kron, 1.0, 8)
    finally:
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)
    ao, ito, _, _ = O.cg(O.kernel_terms(O.KRONECKER), D32, T32, f, s, y, 1.0, 8)
    assert it == ito or n <= 8
    assert rel(a.cpu().numpy(), ao) <= 1e-4


def test_small_engine_c2_matches_multikernel_and_oracle(ctx):
    """GVT_OPT_ENGINE = 4: the whole C2 CG fit (the complete 68 x 442 grid, 100 iterations) in one
    persistent multi-CTA launch with grid barriers.  Auto selects it on C2.  Same fp32 Grams on every
    side: its residual history follows the graph-replayed multi-kernel engine's and the oracle's
    (C2 is ill-conditioned, reading S30, so the weights are compared after 10 iterations, and the
    solver's own in-loop matvec K x_k is checked at the S31 scale); the residual-mode stop equals the
    oracle's iteration count; an ineligible problem is an error."""
    w = synth.config2()
    D = O.gram(w.base, w.Xd, gamma=w.gamma)
    T = O.gram(w.base, w.Xt, gamma=w.gamma)
    Dg, Tg = dev(f32(D)), dev(f32(T))
    kron = G.gvt_kernel_terms(G.KRONECKER)
    f, s, y = dev(w.train_first), dev(w.train_second), dev(w.y)
    D32, T32 = f32(D).astype(np.float64), f32(T).astype(np.float64)
    try:
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)
        ctx.reset_stats()
        a, it, hist, code = ctx.fit(Dg, Tg, f, s, y, kron, w.lam, w.iters)
        st = ctx.stats()
        assert st["last_engine"] == 4 and st["kinds"]["tiny_cg"]["count"] == 1 and code == G.OK and it == w.iters
        # 10 iterations: weights vs the oracle's fp64 CG on the same fp32 Grams and vs the multi-kernel engine
        ao, _, hist_o, _ = O.cg(O.kernel_terms(O.KRONECKER), D32, T32, w.train_first, w.train_second, w.y, w.lam, 10)
        a4, _, h4, _ = ctx.fit(Dg, Tg, f, s, y, kron, w.lam, 10)
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_DENSE)
        a2, _, h2, _ = ctx.fit(Dg, Tg, f, s, y, kron, w.lam, 10)
        assert rel(a4.cpu().numpy(), ao) <= 1e-4 and rel(a4.cpu().numpy(), a2.cpu().numpy()) <= 1e-4
        assert np.allclose(h4, hist_o, rtol=1e-3, atol=1e-9) and np.allclose(h4, h2, rtol=1e-3, atol=1e-9)
        # the in-loop matvec on the final iterate (S31 normalisation, as test_in_loop_matvec_parity)
        x = a.cpu().numpy().astype(np.float64)
        idx = synth.sample_indices(4, w.n, 512)
        ref = O.gvt_matvec(O.kernel_terms(O.KRONECKER), D32, T32, w.train_first[idx], w.train_second[idx],
                           w.train_first, w.train_second, x)
        scale = O.gvt_matvec(O.kernel_terms(O.KRONECKER), np.abs(D32), np.abs(T32), w.train_first[idx],
                             w.train_second[idx], w.train_first, w.train_second, np.abs(x))
        u = ctx.matvec(Dg, Tg, f, s, f, s, a, kron).cpu().numpy()
        assert np.linalg.norm(u[idx] - ref) / np.linalg.norm(scale) <= 1e-5
        # residual-mode stop (a tolerance the oracle's history reaches at iteration 6; C2's residual is
        # not monotone, reading S15)
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_SMALL)
        tol = float(hist_o[6]) * (1 + 1e-9)
        _, it3, h3, _ = ctx.fit(Dg, Tg, f, s, y, kron, w.lam, 200, rel_tol=tol)
        _, it3o, _, _ = O.cg(O.kernel_terms(O.KRONECKER), D32, T32, w.train_first, w.train_second, w.y, w.lam, 200,
                             rel_tol=tol)
        assert it3o <= 6 and abs(it3 - it3o) <= 1 and h3[-1] <= tol
        # determinism: the same bits twice
        b1, _, _, _ = ctx.fit(Dg, Tg, f, s, y, kron, w.lam, 30)
        b2, _, _, _ = ctx.fit(Dg, Tg, f, s, y, kron, w.lam, 30)
        assert torch.equal(b1, b2)
        # an ineligible problem (homogeneous Symmetric) is an error, not a fallback
        with pytest.raises(G.GvtError) as e:
            ctx.fit(Dg, None, f, dev(w.train_first), y, G.gvt_kernel_terms(G.SYMMETRIC), w.lam, 3)
        assert e.value.code == G.E_PARAM
    finally:
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)


@pytest.mark.parametrize("m,q,n", [(3, 5, 7), (70, 300, 10_000), (60, 400, 24_000), (33, 600, 20_000)])
def test_small_engine_shapes(ctx, m, q, n):
    """Ragged shapes through the persistent solver (duplicates, tiles with padding rows, n not a
    multiple of the grid) against the oracle's CG on the same fp32 inputs."""
    rng = np.random.default_rng(m * 7 + n)
    D32 = f32(O.gram(G.BASE_GAUSSIAN, rng.standard_normal((m, 4)), gamma=0.25))
    T32 = f32(O.gram(G.BASE_GAUSSIAN, rng.standard_normal((q, 4)), gamma=0.25))
    f = rng.integers(0, m, n).astype(np.int32)
    s = rng.integers(0, q, n).astype(np.int32)
    y = rng.standard_normal(n).astype(np.float32)
    kron = G.gvt_kernel_terms(G.KRONECKER)
    ctx.set_option(G.OPT_ENGINE, G.ENGINE_SMALL)
    try:
        a, it, _, _ = ctx.fit(dev(D32), dev(T32), dev(f), dev(s), dev(y), kron, 1.0, 8)
        assert ctx.stats()["last_engine"] == 4
    finally:
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)
    ao, ito, _, _ = O.cg(O.kernel_terms(O.KRONECKER), D32, T32, f, s, y, 1.0, 8)
    assert it == ito or n <= 8
    assert rel(a.cpu().numpy(), ao) <= 1e-4


@pytest.mark.parametrize("kernel", [G.KRONECKER, G.SYMMETRIC, G.ANTISYMMETRIC, G.CARTESIAN])
@pytest.mark.parametrize("n", [1, 5, 1185, 30011])
def test_dense_fused_tail_ragged_vs_oracle(ctx, kernel, n):
    """The fused dense-engine CG tail (tail.cu: split-K combine, CG step, next pair matrix in one launch) on ragged
    sizes with duplicate pairs: 8 CG iterations on the tensor-core engine against the oracle's CG, within 1e-4 or 3x
    the sparse engine's own error on the same instance; the profiled launch count shows one CG launch per
    iteration (the tail) instead of three."""
    hom = kernel in HOM
    rng = np.random.default_rng(7 * n + kernel)
    m, q = 37, 29
    D32 = f32(O.gram(G.BASE_GAUSSIAN, rng.standard_normal((m, 4)), gamma=0.25))
    T32 = None if hom else f32(O.gram(G.BASE_GAUSSIAN, rng.standard_normal((q, 4)), gamma=0.25))
    f = rng.integers(0, m, n).astype(np.int32)
    s = rng.integers(0, m if hom else q, n).astype(np.int32)
    y = rng.standard_normal(n).astype(np.float32)
    terms = G.gvt_kernel_terms(kernel)
    args = (dev(D32), None if hom else dev(T32), dev(f), dev(s), dev(y), terms, 1.0, 8)
    try:
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_DENSE)
        ctx.set_option(G.OPT_PROFILE, 1)
        ctx.reset_stats()
        a, it, _, code = ctx.fit(*args)
        k = ctx.stats()["kinds"]
        ctx.set_option(G.OPT_PROFILE, 0)
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_SPARSE)
        asp, _, _, _ = ctx.fit(*args)
    finally:
        ctx.set_option(G.OPT_PROFILE, 0)
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)
    ao, ito, _, _ = O.cg(O.kernel_terms(kernel), D32, T32, f, s, y, 1.0, 8)
    assert code == G.OK and (it == ito or n <= 8)
    assert k["cg_vector"]["count"] <= 8 + 3  # (init, 8 tails -- halted ones return at once --, the direction copy)
    assert np.all(np.isfinite(a.cpu().numpy()))
    assert rel(a.cpu().numpy(), ao) <= max(1e-4, 3 * rel(asp.cpu().numpy(), ao))


@pytest.mark.parametrize("kernel", [G.KRONECKER, G.CARTESIAN])
def test_dense_fused_tail_breakdown(ctx, kernel):
    """CG breakdown inside the fused dense tail: a negative-definite 'Gram' with lambda = 0 makes p^T A p < 0 at the
    first iteration; the tail sets the breakdown flag before touching x, so the fit returns E_BREAKDOWN after 0
    iterations with a = 0 -- the oracle's exit (test_oracle_pins.py::test_cg_breakdown_on_indefinite_operator)."""
    m, q, n = 37, 29, 200
    rng = np.random.default_rng(11 + kernel)
    negD = dev(-np.eye(m, dtype=np.float32))
    negT = dev(-np.eye(q, dtype=np.float32)) if kernel == G.CARTESIAN else dev(np.eye(q, dtype=np.float32))
    cells = rng.choice(m * q, n, replace=False)
    f, s = dev((cells // q).astype(np.int32)), dev((cells % q).astype(np.int32))
    y = dev(rng.standard_normal(n).astype(np.float32))
    try:
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_DENSE)
        a, it, _, code = ctx.fit(negD, negT, f, s, y, G.gvt_kernel_terms(kernel), 0.0, 5, raise_on_breakdown=False)
        st = ctx.stats()
    finally:
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)
    assert st["last_engine"] == 2
    assert code == G.E_BREAKDOWN and it == 0 and np.all(a.cpu().numpy() == 0)
