"""GPU parity of novel-object prediction (NEXT-1; Settings 2-4) through the C ABI:
cross-Grams (gvt_gram_cross) and the GVT on rectangular factors (gvt_matvec_rect,
pairwise_predict_rect) against the oracle's O9 definitions on the same seeded inputs.
Tolerances: Gram max error <= 1e-6 of max |entry|; matvec relative L2 <= 1e-5; the variant
choice and op counts are integers and must be equal."""
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
K_RECT = [G.LINEAR, G.POLY2D, G.GAUSSIAN, G.KRONECKER, G.SYMMETRIC, G.ANTISYMMETRIC, G.RANKING, G.MLPK]


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


@pytest.fixture(params=[G.ENGINE_SPARSE, G.ENGINE_DENSE], ids=["sparse", "dense"])
def engine_ctx(request, ctx):
    ctx.set_option(G.OPT_ENGINE, request.param)
    yield ctx
    ctx.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)


@pytest.mark.parametrize("kind", [G.BASE_LINEAR, G.BASE_GAUSSIAN, G.BASE_POLY])
@pytest.mark.parametrize("gram_engine", [1, 0], ids=["simt", "tc"])
def test_gram_cross_parity(ctx, kind, gram_engine):
    """k(X_i, Y_j) for two different tables, ragged sizes across tiles."""
    ctx.set_option(G.OPT_GRAM_ENGINE, gram_engine)
    try:
        rng = np.random.default_rng(70 + kind)
        for m, m2, dim in [(1, 3, 5), (300, 77, 37), (129, 517, 128)]:
            X = rng.standard_normal((m, dim)).astype(np.float32)
            Y = rng.standard_normal((m2, dim)).astype(np.float32)
            K = ctx.gram_cross(kind, dev(X), dev(Y), gamma=1.0 / dim).cpu().numpy()
            ref = O.gram(kind, X, Y, gamma=1.0 / dim)
            assert K.shape == (m, m2)
            assert np.abs(K - ref).max() <= 1e-6 * np.abs(ref).max(), (m, m2, dim)
    finally:
        ctx.set_option(G.OPT_GRAM_ENGINE, 0)


def _rect_instance(seed, kernel, mo, mi, qo, qi, n_out, n_in, dim=12):
    hom = kernel in HOM
    rng = np.random.default_rng(seed)
    Xtr, Xte = rng.standard_normal((mi, dim)), rng.standard_normal((mo, dim))
    Dx = O.gram(O.BASE_GAUSSIAN, Xte, Xtr, gamma=1.0 / dim)
    Tx = None
    if not hom:
        Ytr, Yte = rng.standard_normal((qi, dim)), rng.standard_normal((qo, dim))
        Tx = O.gram(O.BASE_GAUSSIAN, Yte, Ytr, gamma=1.0 / dim)
    else:
        qo, qi = mo, mi
    inf, ins = rng.integers(0, mi, n_in).astype(np.int32), rng.integers(0, qi, n_in).astype(np.int32)
    of, os_ = rng.integers(0, mo, n_out).astype(np.int32), rng.integers(0, qo, n_out).astype(np.int32)
    a = rng.standard_normal(n_in).astype(np.float32)
    return f32(Dx), f32(Tx), of, os_, inf, ins, a


@pytest.mark.parametrize("kernel", K_RECT)
def test_matvec_rect_vs_oracle(engine_ctx, kernel):
    """Every kernel but Cartesian on cross-Grams: small ragged shapes and a medium one (several
    tiles, m_out != m_in, q_out != q_in) against the oracle's rectangular definition."""
    terms = G.gvt_kernel_terms(kernel)
    shapes = [(3, 5, 4, 2, 7, 11), (1, 1, 1, 1, 1, 1), (9, 4, 6, 8, 0, 13), (150, 300, 90, 200, 5000, 20000)]
    for i, (mo, mi, qo, qi, no, ni) in enumerate(shapes):
        Dx, Tx, of, os_, inf, ins, a = _rect_instance(100 * kernel + i, kernel, mo, mi, qo, qi, no, ni)
        u, v, ops = engine_ctx.matvec_rect(dev(Dx), None if Tx is None else dev(Tx), dev(of), dev(os_), dev(inf),
                                           dev(ins), dev(a), terms)
        ref = O.explicit_rect_matvec(kernel, Dx, Tx, of, os_, inf, ins, a)
        assert u.shape[0] == no
        if no:
            assert rel(u.cpu().numpy(), ref) <= 1e-5, (kernel, i, rel(u.cpu().numpy(), ref))


def test_matvec_rect_variants_and_costs(engine_ctx):
    """Kronecker on cross-Grams: variants 1 and 2 give the same u; auto picks the cheaper variant
    by Theorem 1's cost exactly as the oracle does (SPEC gvt_cost, ties -> 1) -- both ways
    round -- and reports the same op count."""
    kron = G.gvt_kernel_terms(G.KRONECKER)
    # (m_out, m_in, q_out, q_in): few novel drugs, many target rows -> variant 2 is cheaper, and the mirror
    for mo, mi, qo, qi in [(4, 300, 250, 40), (250, 40, 4, 300), (50, 50, 50, 50)]:
        Dx, Tx, of, os_, inf, ins, a = _rect_instance(mo * 7 + qi, G.KRONECKER, mo, mi, qo, qi, 3000, 8000)
        ref, ov, oops = O.gvt_rect(Dx, Tx, of, os_, inf, ins, a, 0)
        outs = {}
        for var in (0, 1, 2):
            u, v, ops = engine_ctx.matvec_rect(dev(Dx), dev(Tx), dev(of), dev(os_), dev(inf), dev(ins), dev(a), kron,
                                               variant=var)
            outs[var] = (u.cpu().numpy(), v, ops)
            assert rel(outs[var][0], ref) <= 1e-5, (mo, var)
        assert (outs[0][1], outs[0][2]) == (ov, oops)
        _, v1, ops1 = O.gvt_rect(Dx, Tx, of, os_, inf, ins, a, 1)
        _, v2, ops2 = O.gvt_rect(Dx, Tx, of, os_, inf, ins, a, 2)
        assert (outs[1][1], outs[1][2], outs[2][1], outs[2][2]) == (1, ops1, 2, ops2)
    assert ov == 1  # the square case ties -> variant 1


def test_settings_2_to_4_end_to_end(ctx):
    """Settings 2-4 on C1: fit on the training objects (square Grams), then predict pairs with a
    novel drug, a novel target, or both, from cross-Grams built on the GPU from the new objects'
    features.  Equals the square path over the union object table (the cross-Grams are its
    sub-blocks) and the oracle's rectangular definition on the oracle's weights."""
    w = synth.config1()
    rng = np.random.default_rng(9)
    kron = G.gvt_kernel_terms(G.KRONECKER)
    Xd_new = rng.standard_normal((7, w.Xd.shape[1])).astype(np.float32)
    Xt_new = rng.standard_normal((9, w.Xt.shape[1])).astype(np.float32)
    D = ctx.gram(w.base, dev(w.Xd), gamma=w.gamma)
    T = ctx.gram(w.base, dev(w.Xt), gamma=w.gamma)
    a, it, _, _ = ctx.fit(D, T, dev(w.train_first), dev(w.train_second), dev(w.y), kron, w.lam, w.iters)
    Do = O.gram(w.base, w.Xd, gamma=w.gamma)
    To = O.gram(w.base, w.Xt, gamma=w.gamma)
    ao, _, _, _ = O.cg(O.kernel_terms(O.KRONECKER), Do, To, w.train_first, w.train_second, w.y, w.lam, w.iters)
    n = 400
    for setting in (2, 3, 4):
        Xd_out = w.Xd if setting == 2 else Xd_new   # setting 2: known drugs, novel targets
        Xt_out = w.Xt if setting == 3 else Xt_new   # setting 3: novel drugs, known targets
        Dx = ctx.gram_cross(w.base, dev(Xd_out), dev(w.Xd), gamma=w.gamma)
        Tx = ctx.gram_cross(w.base, dev(Xt_out), dev(w.Xt), gamma=w.gamma)
        tf = rng.integers(0, Xd_out.shape[0], n).astype(np.int32)
        ts = rng.integers(0, Xt_out.shape[0], n).astype(np.int32)
        sc = ctx.predict_rect(Dx, Tx, dev(tf), dev(ts), dev(w.train_first), dev(w.train_second), a, kron)
        sc = sc.cpu().numpy()
        ref = O.explicit_rect_matvec(O.KRONECKER, O.gram(w.base, Xd_out, w.Xd, gamma=w.gamma),
                                     O.gram(w.base, Xt_out, w.Xt, gamma=w.gamma), tf, ts, w.train_first,
                                     w.train_second, ao)
        assert np.abs(sc - ref).max() <= 1e-4, setting
        # the square path over the union table gives the same scores
        Du = ctx.gram(w.base, dev(np.vstack([w.Xd, Xd_out])), gamma=w.gamma)
        Tu = ctx.gram(w.base, dev(np.vstack([w.Xt, Xt_out])), gamma=w.gamma)
        su = ctx.predict(Du, Tu, dev(tf + w.m), dev(ts + w.q), dev(w.train_first), dev(w.train_second), a, kron)
        assert rel(sc, su.cpu().numpy()) <= 1e-5, setting


def test_rect_errors(ctx):
    Dx, Tx, of, os_, inf, ins, a = _rect_instance(1, G.KRONECKER, 3, 4, 5, 6, 10, 10)
    with pytest.raises(G.GvtError) as e:
        ctx.matvec_rect(dev(Dx), dev(Tx), dev(of), dev(os_), dev(inf), dev(ins), dev(a),
                        G.gvt_kernel_terms(G.CARTESIAN))
    assert e.value.code == G.E_KERNEL
    bad = of.copy()
    bad[0] = 3
    with pytest.raises(G.GvtError) as e:
        ctx.matvec_rect(dev(Dx), dev(Tx), dev(bad), dev(os_), dev(inf), dev(ins), dev(a), G.gvt_kernel_terms(G.KRONECKER))
    assert e.value.code == G.E_INDEX
    with pytest.raises(G.GvtError) as e:
        ctx.matvec_rect(dev(Dx), dev(Tx), dev(of), dev(os_), dev(inf), dev(ins), dev(a),
                        G.gvt_kernel_terms(G.POLY2D), variant=2)
    assert e.value.code == G.E_PARAM


# ----------------------------------------------------------------------------- Tanimoto (NEXT-4)
def test_tanimoto_gram_parity(ctx):
    """Tanimoto Gram (bit-packed popcounts) vs the oracle's min/max definition: fingerprint-like
    densities 1-30 %, all-zero rows (T1), lengths across word and tile boundaries (Heterodimer's
    2554 + 768 + 83 = 3405 bits), square and cross forms; exactly 1 on the square diagonal."""
    rng = np.random.default_rng(77)
    for m, m2, dim in [(1, 1, 1), (65, 33, 31), (300, 129, 3405), (517, 64, 881)]:
        X = (rng.uniform(size=(m, dim)) < rng.uniform(0.01, 0.3, size=(m, 1))).astype(np.float32)
        Y = (rng.uniform(size=(m2, dim)) < 0.05).astype(np.float32)
        X[0] = 0
        Y[-1] = 0
        K = ctx.gram(G.BASE_TANIMOTO, dev(X)).cpu().numpy()
        ref = O.gram(O.BASE_TANIMOTO, X)
        assert np.abs(K - ref).max() <= 1e-6, (m, dim)
        assert np.all(np.diag(K) == 1.0)
        Kx = ctx.gram_cross(G.BASE_TANIMOTO, dev(X), dev(Y)).cpu().numpy()
        assert np.abs(Kx - O.gram(O.BASE_TANIMOTO, X, Y)).max() <= 1e-6, (m, m2, dim)
    with pytest.raises(G.GvtError) as e:
        ctx.gram(G.BASE_TANIMOTO, dev(np.array([[0.0, 0.5]], np.float32)))
    assert e.value.code == G.E_PARAM


def test_tanimoto_symmetric_kernel_fit(ctx):
    """A Heterodimer-shaped homogeneous problem (proteins with binary
    domain / phylogenetic / localisation features, Tanimoto base kernel, symmetric pairwise
    kernel; synthetic stand-in): GPU Gram + 20 CG iterations match the oracle's weights."""
    rng = np.random.default_rng(78)
    m, dim, n = 300, 3405, 1500
    X = (rng.uniform(size=(m, dim)) < rng.uniform(0.002, 0.05, size=(m, 1))).astype(np.float32)
    f = rng.integers(0, m, n).astype(np.int32)
    s = rng.integers(0, m, n).astype(np.int32)
    y = np.sign(rng.standard_normal(n)).astype(np.float32)
    sym = G.gvt_kernel_terms(G.SYMMETRIC)
    D = ctx.gram(G.BASE_TANIMOTO, dev(X))
    a, it, _, _ = ctx.fit(D, None, dev(f), dev(s), dev(y), sym, 1.0, 20)
    Do = O.gram(O.BASE_TANIMOTO, X)
    ao, _, _, _ = O.cg(O.kernel_terms(O.SYMMETRIC), Do, None, f, s, y, 1.0, 20)
    assert rel(a.cpu().numpy(), ao) <= 1e-4
