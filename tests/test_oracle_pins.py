"""Pins for the fp64 oracle (-m "not gpu").

Each test pins an oracle function to something OTHER than the oracle itself:
values printed in the paper or SPEC (tests/golden, cited), closed forms evaluated by
library routines (numpy matmul / kron, scipy cdist, numpy.linalg.solve), the
paper's operator algebra (P, Q from Definition 1, the Corollary operators, Theorem 2,
Table 4a feature maps), invariants and brute force on tiny inputs.  A plausible
mistake (dropped term, wrong sign, transposed operand, wrong selector) fails one.
"""
import itertools
import json

import numpy as np
import pytest
from scipy.spatial.distance import cdist

import oracle as O
import synth
from conftest import golden_path, load_golden_matrix

K_ALL = [O.LINEAR, O.POLY2D, O.GAUSSIAN, O.KRONECKER, O.SYMMETRIC, O.ANTISYMMETRIC, O.RANKING, O.MLPK,
         O.CARTESIAN]
HET = [O.LINEAR, O.POLY2D, O.GAUSSIAN, O.KRONECKER, O.CARTESIAN]
HOM = [O.SYMMETRIC, O.ANTISYMMETRIC, O.RANKING, O.MLPK]
SPEC = json.load(open(golden_path("spec_worked_values.json")))


def rel(x, ref):
    x, ref = np.asarray(x, float), np.asarray(ref, float)
    nr = np.linalg.norm(ref)
    return np.linalg.norm(x - ref) / (nr if nr > 1e-30 else 1.0)


# ----------------------------------------------------------------------------- base Grams
def test_gram_spec_worked_values():
    g = SPEC["linear_base"]
    assert O.gram(O.BASE_LINEAR, g["X"], g["Y"])[0, 0] == 11.0
    g = SPEC["gaussian_base"]
    assert O.gram(O.BASE_GAUSSIAN, g["X"], g["Y"], gamma=g["gamma"])[0, 0] == pytest.approx(np.exp(-1.0), abs=1e-15)


def test_gram_matches_library_closed_forms():
    rng = np.random.default_rng(0)
    X, Y = rng.standard_normal((13, 7)), rng.standard_normal((9, 7))
    assert np.abs(O.gram(O.BASE_LINEAR, X, Y) - X @ Y.T).max() < 1e-12
    gam = 0.37
    ref = np.exp(-gam * cdist(X, Y, "sqeuclidean"))
    assert np.abs(O.gram(O.BASE_GAUSSIAN, X, Y, gamma=gam) - ref).max() < 1e-13
    ref = (0.2 * (X @ Y.T) + 1.5) ** 3
    assert np.abs(O.gram(O.BASE_POLY, X, Y, gamma=0.2, coef0=1.5, degree=3) - ref).max() < 1e-10


def test_gram_gaussian_diag_exact_and_psd():
    X = synth.config1().Xd
    K = O.gram(O.BASE_GAUSSIAN, X, gamma=1 / 16)
    assert np.all(np.diag(K) == 1.0)                       # SPEC.md:201, reading S29
    ev = np.linalg.eigvalsh(K)
    assert ev.min() >= -1e-10 * ev.max()                    # PSD
    assert np.abs(K - K.T).max() == 0.0


def test_gram_rejects_bad_gamma():
    with pytest.raises(O.OracleError) as e:
        O.gram(O.BASE_GAUSSIAN, [[0.0]], gamma=0.0)
    assert e.value.code == O.E_PARAM


# ----------------------------------------------------------------------------- kernel values
def test_kernel_value_spec_worked_values():
    kv = SPEC["kernel_value"]
    D, T = np.array([[kv["D00"]]]), np.array([[kv["T00"]]])
    assert O.kernel_value(O.LINEAR, D, T, (0, 0), (0, 0)) == kv["linear"]
    assert O.kernel_value(O.POLY2D, D, T, (0, 0), (0, 0)) == kv["poly2d"]
    assert O.kernel_value(O.KRONECKER, D, T, (0, 0), (0, 0)) == 6.0
    rng = np.random.default_rng(1)
    F = rng.standard_normal((4, 3))
    Dh = F @ F.T
    for dd in range(4):   # MLPK / Ranking / Anti vanish on a self pair (S18)
        for b in itertools.product(range(4), repeat=2):
            assert abs(O.kernel_value(O.MLPK, Dh, None, (dd, dd), b)) < 1e-28
            assert abs(O.kernel_value(O.RANKING, Dh, None, (dd, dd), b)) < 1e-14
            assert abs(O.kernel_value(O.ANTISYMMETRIC, Dh, None, (dd, dd), b)) < 1e-14


def _feature_map(kernel, fd, ft, ed=None, et=None):
    """Table 4a: the pair feature maps, written from the table."""
    if kernel == O.LINEAR:
        return np.concatenate([fd, ft])
    if kernel == O.POLY2D:
        c = np.concatenate([fd, ft])
        return np.kron(c, c)
    if kernel in (O.KRONECKER, O.GAUSSIAN):
        return np.kron(fd, ft)
    if kernel == O.SYMMETRIC:
        return np.sqrt(0.5) * (np.kron(fd, ft) + np.kron(ft, fd))
    if kernel == O.ANTISYMMETRIC:
        return np.sqrt(0.5) * (np.kron(fd, ft) - np.kron(ft, fd))
    if kernel == O.RANKING:
        return fd - ft
    if kernel == O.MLPK:
        return np.kron(fd - ft, fd - ft)
    if kernel == O.CARTESIAN:
        return np.concatenate([np.kron(fd, et), np.kron(ed, ft)])
    raise ValueError


@pytest.mark.parametrize("kernel", K_ALL)
def test_kernel_value_equals_feature_map_inner_product(kernel):
    """Table 4a feature maps vs Table 4b kernel values: a sign error (e.g. the
    Corollary's printed (P-I) for Anti-symmetric) or a dropped term fails here."""
    rng = np.random.default_rng(100 + kernel)
    hom = kernel in HOM
    m, q, r = 4, 3, 3
    Fd = rng.standard_normal((m, r))
    Ft = Fd if hom else rng.standard_normal((q, r))
    qq = m if hom else q
    D, T = Fd @ Fd.T, (None if hom else Ft @ Ft.T)
    Id, It = np.eye(m), np.eye(qq)
    for (d, t), (db, tb) in itertools.product(itertools.product(range(m), range(qq)), repeat=2):
        if (d * qq + t) % 3 and (db * qq + tb) % 2:    # thin the 144..256 combos a little
            continue
        phi_o = _feature_map(kernel, Fd[d], Ft[t], Id[d], It[t])
        phi_i = _feature_map(kernel, Fd[db], Ft[tb], Id[db], It[tb])
        assert O.kernel_value(kernel, D, T, (d, t), (db, tb)) == pytest.approx(phi_o @ phi_i, abs=1e-11)


def test_gaussian_pairwise_is_gaussian_on_concatenated_features():
    """exp(-g||(xd,xt)-(xd',xt')||^2) = k_D * k_T (squared norm, S4)."""
    rng = np.random.default_rng(7)
    Xd, Xt, g = rng.standard_normal((5, 3)), rng.standard_normal((4, 2)), 0.3
    D, T = O.gram(O.BASE_GAUSSIAN, Xd, gamma=g), O.gram(O.BASE_GAUSSIAN, Xt, gamma=g)
    for d, t, db, tb in [(0, 1, 2, 3), (4, 0, 4, 0), (1, 3, 0, 2)]:
        direct = np.exp(-g * np.sum((np.concatenate([Xd[d], Xt[t]]) - np.concatenate([Xd[db], Xt[tb]])) ** 2))
        assert O.kernel_value(O.GAUSSIAN, D, T, (d, t), (db, tb)) == pytest.approx(direct, rel=1e-13)


def test_kernel_value_invariants():
    rng = np.random.default_rng(3)
    F = rng.standard_normal((5, 4))
    D = F @ F.T
    for _ in range(50):
        d, dp, db, dbp = rng.integers(0, 5, 4)
        kv = lambda k, o, i: O.kernel_value(k, D, None, o, i)
        # symmetric: invariant to swapping either pair; anti/ranking flip; mlpk invariant
        assert kv(O.SYMMETRIC, (d, dp), (db, dbp)) == pytest.approx(kv(O.SYMMETRIC, (dp, d), (db, dbp)))
        assert kv(O.SYMMETRIC, (d, dp), (db, dbp)) == pytest.approx(kv(O.SYMMETRIC, (d, dp), (dbp, db)))
        assert kv(O.ANTISYMMETRIC, (d, dp), (db, dbp)) == pytest.approx(-kv(O.ANTISYMMETRIC, (dp, d), (db, dbp)))
        assert kv(O.RANKING, (d, dp), (db, dbp)) == pytest.approx(-kv(O.RANKING, (dp, d), (db, dbp)))
        assert kv(O.MLPK, (d, dp), (db, dbp)) == pytest.approx(kv(O.MLPK, (dp, d), (dbp, db)))
        # Poly2D = Linear^2, MLPK = Ranking^2
        assert kv(O.POLY2D, (d, dp), (db, dbp)) == pytest.approx(kv(O.LINEAR, (d, dp), (db, dbp)) ** 2)
        assert kv(O.MLPK, (d, dp), (db, dbp)) == pytest.approx(kv(O.RANKING, (d, dp), (db, dbp)) ** 2)


# ----------------------------------------------------------------------------- P, Q, Corollary
def commutation(nd, nt):
    """Definition 1: P[(t,d),(d',t')] = 1 iff d=d', t=t'."""
    P = np.zeros((nt * nd, nd * nt))
    for t in range(nt):
        for d in range(nd):
            P[t * nd + d, d * nt + t] = 1
    return P


def unification(nd, nt):
    """Definition 1: Q[(d,t),(d',d'')] = 1 iff d=d'=d''."""
    Q = np.zeros((nd * nt, nd * nd))
    for d in range(nd):
        for t in range(nt):
            Q[d * nt + t, d * nd + d] = 1
    return Q


def pq_product(nd, nt):
    """PQ values given in Definition 1: PQ[(d,t),(t',t'')] = 1 iff t=t'=t''."""
    M = np.zeros((nd * nt, nt * nt))
    for d in range(nd):
        for t in range(nt):
            M[d * nt + t, t * nt + t] = 1
    return M


def test_P_Q_match_paper_example():
    assert np.array_equal(commutation(3, 2), load_golden_matrix("paper_P_3drugs_2targets.txt"))
    assert np.array_equal(unification(3, 2), load_golden_matrix("paper_Q_3drugs_2targets.txt"))


def test_theorem2_identities():
    """Theorem 2 checked with explicit matrices."""
    rng = np.random.default_rng(11)
    nd, nt = 3, 4
    Fd, Ft = rng.standard_normal((nd, 2)), rng.standard_normal((nt, 2))
    D, T = Fd @ Fd.T, Ft @ Ft.T
    P = commutation(nd, nt)
    assert np.allclose(P @ P.T, np.eye(nd * nt)) and np.allclose(P.T @ P, np.eye(nd * nt))
    assert np.allclose(P @ np.kron(D, T), np.kron(T, D) @ P)
    assert np.allclose(P @ np.kron(D, T) @ P.T, np.kron(T, D))
    Ph = commutation(nd, nd)
    assert np.array_equal(Ph, Ph.T)
    assert np.allclose(Ph @ np.kron(D, D), np.kron(D, D) @ Ph)
    Q = unification(nd, nt)
    assert np.allclose(Q @ np.kron(D, D) @ Q.T, np.kron(D * D, np.ones((nt, nt))))


def corollary_operator(kernel, D, T):
    """The Corollary table as explicit matrices over the whole domain,
    natural pair order.  Anti-symmetric uses (I-P) (reading S3); MLPK uses (I-Q)^T on the
    right (reading S22)."""
    if kernel in HOM:
        n = D.shape[0]
        P, Q, I, one = commutation(n, n), unification(n, n), np.eye(n * n), np.ones((n, n))
        DD = np.kron(D, D)
        if kernel == O.SYMMETRIC:
            return (P + I) @ DD
        if kernel == O.ANTISYMMETRIC:
            return (I - P) @ DD
        if kernel == O.RANKING:
            return (I - P) @ np.kron(D, one) @ (I - P)
        if kernel == O.MLPK:
            return (I + P) @ (I - Q) @ DD @ (I - Q).T @ (I + P)
    nd, nt = D.shape[0], T.shape[0]
    if kernel == O.LINEAR:
        return np.kron(D, np.ones((nt, nt))) + np.kron(np.ones((nd, nd)), T)
    if kernel == O.POLY2D:
        Q, PQ = unification(nd, nt), pq_product(nd, nt)
        return Q @ np.kron(D, D) @ Q.T + 2 * np.kron(D, T) + PQ @ np.kron(T, T) @ PQ.T
    if kernel in (O.KRONECKER, O.GAUSSIAN):
        return np.kron(D, T)
    if kernel == O.CARTESIAN:
        return np.kron(D, np.eye(nt)) + np.kron(np.eye(nd), T)
    raise ValueError


def sampling_operator(f, s, nd, nt):
    """R(d,t) of PAPER.md:302-310: R[i,(d,t)] = 1 iff (d,t) = (d_i,t_i)."""
    R = np.zeros((len(f), nd * nt))
    R[np.arange(len(f)), np.asarray(f) * nt + np.asarray(s)] = 1
    return R


@pytest.mark.parametrize("kernel", K_ALL)
def test_explicit_matrix_equals_corollary_operator(kernel):
    """Table 4b (the oracle's definition) == R_bar K_op R^T with the Corollary operator."""
    for seed in range(5):
        w = synth.tiny(seed, m=4, q=3, n=10, n_out=7, homogeneous=kernel in HOM)
        D = O.gram(O.BASE_GAUSSIAN, w.Xd, gamma=0.5)
        T = None if w.Xt is None else O.gram(O.BASE_GAUSSIAN, w.Xt, gamma=0.5)
        nt = D.shape[0] if T is None else T.shape[0]
        Kop = corollary_operator(kernel, D, T)
        Rin = sampling_operator(w.train_first, w.train_second, D.shape[0], nt)
        Rout = sampling_operator(w.test_first, w.test_second, D.shape[0], nt)
        Kref = Rout @ Kop @ Rin.T
        K = O.explicit_matrix(kernel, D, T, w.test_first, w.test_second, w.train_first, w.train_second)
        assert np.abs(K - Kref).max() < 1e-12


def test_printed_antisymmetric_sign_is_negative_semidefinite():
    """Reading S3: the Corollary's printed (P-I)(D(x)D) is NSD on the full domain, so it
    cannot be the kernel of Table 4b; (I-P)(D(x)D) is PSD."""
    rng = np.random.default_rng(5)
    F = rng.standard_normal((4, 4))
    D = F @ F.T
    n = 4
    P, I = commutation(n, n), np.eye(n * n)
    ev_printed = np.linalg.eigvalsh((P - I) @ np.kron(D, D))
    ev_used = np.linalg.eigvalsh((I - P) @ np.kron(D, D))
    assert ev_printed.max() <= 1e-10 and ev_printed.min() < -1e-3
    assert ev_used.min() >= -1e-10


# ----------------------------------------------------------------------------- term lists
def test_term_counts_and_mlpk_coefficients():
    tc = SPEC["term_counts"]
    for name, k in zip(synth.KERNEL_NAMES, range(9)):
        assert len(O.kernel_terms(k)) == tc[name], name
    assert [t.coef for t in O.kernel_terms(O.MLPK)] == SPEC["mlpk_coefficients"]["coefs"]
    with pytest.raises(O.OracleError):
        O.kernel_terms(42)


def eval_term_python(t, D, T, o, i):
    """The KernelTerm meaning: coef * L[rl(o), cl(i)] * R[rr(o), cr(i)]."""
    coef, left, right, rl, rr, cl, cr = t.as_tuple()
    Tm = D if T is None else T

    def fv(kind, r, c):
        return {O.DRUG: lambda: D[r, c], O.TARGET: lambda: Tm[r, c], O.ONES: lambda: 1.0,
                O.IDENTITY: lambda: float(r == c)}[kind]()
    return coef * fv(left, o[rl], i[cl]) * fv(right, o[rr], i[cr])


@pytest.mark.parametrize("kernel", K_ALL)
def test_term_assembly_equals_table4b(kernel):
    """Decomposition soundness: summing the Corollary terms entrywise
    reproduces the Table 4b value of every argument pair."""
    w = synth.tiny(3, m=4, q=3, homogeneous=kernel in HOM)
    D = O.gram(O.BASE_GAUSSIAN, w.Xd, gamma=0.5)
    T = None if w.Xt is None else O.gram(O.BASE_GAUSSIAN, w.Xt, gamma=0.5)
    qq = D.shape[0] if T is None else T.shape[0]
    terms = O.kernel_terms(kernel)
    for o in itertools.product(range(4), range(qq)):
        for i in itertools.product(range(4), range(qq)):
            v = sum(eval_term_python(t, D, T, o, i) for t in terms)
            assert v == pytest.approx(O.kernel_value(kernel, D, T, o, i), abs=1e-12)


# ----------------------------------------------------------------------------- GVT exactness
@pytest.mark.parametrize("kernel", K_ALL)
def test_gvt_equals_explicit_on_200_tiny_instances(kernel):
    """Theorem 1 is exact: the per-term GVT (both variants and auto)
    equals the explicit product within 1e-12 relative on
    out != in samples with duplicate and self pairs."""
    terms = O.kernel_terms(kernel)
    hom = kernel in HOM
    for seed in range(200):
        rng = np.random.default_rng(seed)
        m, q = int(rng.integers(1, 7)), int(rng.integers(1, 7))
        w = synth.tiny(seed, m=m, q=q, n=int(rng.integers(0, 20)), n_out=int(rng.integers(0, 15)),
                       homogeneous=hom)
        D = O.gram(O.BASE_GAUSSIAN, w.Xd, gamma=0.5)
        T = None if w.Xt is None else O.gram(O.BASE_GAUSSIAN, w.Xt, gamma=0.5)
        a = synth.random_vector(seed, w.n)
        ref = O.explicit_matvec(kernel, D, T, w.test_first, w.test_second, w.train_first, w.train_second, a)
        for variant in (1, 2, 0):
            u = O.gvt_matvec(terms, D, T, w.test_first, w.test_second, w.train_first, w.train_second, a,
                             variant=variant)
            assert rel(u, ref) <= 1e-12 or np.abs(u - ref).max() < 1e-13, (seed, variant)


def test_gvt_spec_small_cases():
    g = SPEC["gvt_single"]
    kron = O.kernel_terms(O.KRONECKER)
    u = O.gvt_matvec(kron, [[g["A"]]], [[g["B"]]], [0], [0], [0], [0], [g["v"]])
    assert u[0] == g["u"]
    # identity Kronecker over the full grid returns v
    f, s = np.repeat(np.arange(2), 2), np.tile(np.arange(2), 2)
    v = np.array([0.3, -1.2, 2.5, 7.0])
    assert np.array_equal(O.gvt_matvec(kron, np.eye(2), np.eye(2), f, s, f, s, v), v)
    # empty samples are legal
    assert O.gvt_matvec(kron, np.eye(2), np.eye(2), [], [], f, s, v).shape == (0,)
    assert np.array_equal(O.gvt_matvec(kron, np.eye(2), np.eye(2), f, s, [], [], []), np.zeros(4))


def test_gvt_cost_and_op_count_spec_example():
    """costs 17 / 14 and the FMA counter of variant 1."""
    c = SPEC["gvt_cost"]
    # out sample: 3 pairs over 2 drugs, 2 targets; in sample: 4 pairs over 3 drugs, 2 targets
    of, os_ = [0, 1, 1], [0, 1, 0]
    inf, ins = [0, 1, 2, 2], [0, 1, 1, 0]
    term = O.kernel_terms(O.KRONECKER)[0]
    c1, c2 = O.term_cost(term, 3, 2, False, of, os_, inf, ins)
    assert (c1, c2) == (c["cost1"], c["cost2"])
    D, T = np.eye(3), np.eye(2)
    _, ops1 = O.term_gvt(term, D, T, of, os_, inf, ins, np.ones(4), variant=1)
    _, ops2 = O.term_gvt(term, D, T, of, os_, inf, ins, np.ones(4), variant=2)
    assert (ops1, ops2) == (c["cost1"], c["cost2"])
    _, ops_auto = O.gvt_matvec([term], D, T, of, os_, inf, ins, np.ones(4), variant=0, return_ops=True)
    assert ops_auto == min(c1, c2)


def test_roth_vec_trick_complete_grid():
    """PAPER.md:324 (Roth's column lemma): on the complete grid, the Kronecker matvec is
    U = D A T^T with A the m x q reshape of a -- checked against numpy matmul."""
    w = synth.config2()
    Xd, Xt = w.Xd.astype(np.float64), w.Xt.astype(np.float64)
    D, T = Xd @ Xd.T, Xt @ Xt.T
    a = synth.random_vector(0, w.n).astype(np.float64)
    u = O.gvt_matvec(O.kernel_terms(O.KRONECKER), D, T, w.train_first, w.train_second, w.train_first,
                     w.train_second, a)
    U = D @ a.reshape(68, 442) @ T.T
    assert rel(u, U.reshape(-1)) < 1e-12


def test_ranking_equals_oriented_incidence():
    """the Ranking kernel matrix is M^T D M with the oriented
    incidence operator M."""
    w = synth.tiny(9, m=6, n=15, n_out=15, homogeneous=True)
    D = O.gram(O.BASE_GAUSSIAN, w.Xd, gamma=0.5)
    M = np.zeros((6, w.n))
    M[w.train_first, np.arange(w.n)] += 1
    M[w.train_second, np.arange(w.n)] -= 1
    K = O.explicit_matrix(O.RANKING, D, None, w.train_first, w.train_second, w.train_first, w.train_second)
    assert np.abs(K - M.T @ D @ M).max() < 1e-12


def test_gvt_linearity_and_psd():
    w = synth.tiny(4, m=5, n=14, n_out=14, homogeneous=True)
    D = O.gram(O.BASE_GAUSSIAN, w.Xd, gamma=0.5)
    for k in HOM:
        terms = O.kernel_terms(k)
        a, b = synth.random_vector(1, w.n).astype(np.float64), synth.random_vector(2, w.n).astype(np.float64)
        f, s = w.train_first, w.train_second
        lhs = O.gvt_matvec(terms, D, None, f, s, f, s, 2.0 * a - 3.0 * b)
        rhs = 2.0 * O.gvt_matvec(terms, D, None, f, s, f, s, a) - 3.0 * O.gvt_matvec(terms, D, None, f, s, f, s, b)
        assert rel(lhs, rhs) < 1e-12
        K = O.explicit_matrix(k, D, None, f, s, f, s)
        ev = np.linalg.eigvalsh(0.5 * (K + K.T))
        assert ev.min() >= -1e-10 * max(1.0, ev.max())


def test_homogeneity_errors():
    D = np.eye(3)
    with pytest.raises(O.OracleError) as e:
        O.explicit_matvec(O.SYMMETRIC, D, np.eye(2), [0], [0], [0], [0], [1.0])
    assert e.value.code == O.E_HOMOGENEOUS
    with pytest.raises(O.OracleError) as e:
        O.explicit_matvec(O.KRONECKER, D, np.eye(2), [0], [2], [0], [0], [1.0])
    assert e.value.code == O.E_INDEX


# ----------------------------------------------------------------------------- CG
def test_cg_scalar_systems():
    # (2 I) a = y after one iteration (K = I via identity Grams on the full grid, lambda = 1)
    f, s = np.repeat(np.arange(3), 2), np.tile(np.arange(2), 3)
    y = np.array([1.0, -2.0, 0.5, 4.0, 3.0, -1.0])
    kron = O.kernel_terms(O.KRONECKER)
    x, it, hist, rc = O.cg(kron, np.eye(3), np.eye(2), f, s, y, 1.0, 5)
    assert rc == O.OK and it == 1 and np.allclose(x, y / 2, atol=1e-15)
    # y = 0 -> a = 0, zero iterations
    x, it, hist, rc = O.cg(kron, np.eye(3), np.eye(2), f, s, np.zeros(6), 1.0, 5)
    assert it == 0 and np.all(x == 0)
    # single pair ridge
    r = SPEC["ridge_single_pair"]
    x, it, _, rc = O.cg(kron, [[r["D"]]], [[r["T"]]], [0], [0], [r["y"]], r["lambda"], 3)
    assert x[0] == pytest.approx(r["a"], abs=1e-15)
    # lambda = 0, K = I -> a = y
    x, it, _, _ = O.cg(kron, np.eye(3), np.eye(2), f, s, y, 0.0, 5)
    assert np.allclose(x, y, atol=1e-15)


def test_cg_matches_dense_direct_solve_on_C1():
    """On C1 (kappa ~ 40) 50 fp64 iterations converge: the oracle's weights equal
    numpy.linalg.solve of the explicit system (K + lambda I) a = y within 1e-10, the
    recursive relres is <= 1e-6, and the A-norm error is non-increasing (reading S15)."""
    w = synth.config1()
    D = O.gram(O.BASE_GAUSSIAN, w.Xd, gamma=w.gamma)
    T = O.gram(O.BASE_GAUSSIAN, w.Xt, gamma=w.gamma)
    f, s = w.train_first, w.train_second
    K = O.explicit_matrix(O.KRONECKER, D, T, f, s, f, s)
    A = K + w.lam * np.eye(w.n)
    xs = np.linalg.solve(A, w.y.astype(np.float64))
    kron = O.kernel_terms(O.KRONECKER)
    x, it, hist, rc = O.cg(kron, D, T, f, s, w.y, w.lam, w.iters)
    assert rc == O.OK and it == 50
    assert rel(x, xs) < 1e-10
    assert hist[-1] <= 1e-6
    errs = []
    for k in range(1, 25):
        xk, _, _, _ = O.cg(kron, D, T, f, s, w.y, w.lam, k)
        e = xk - xs
        errs.append(np.sqrt(e @ A @ e))
    assert all(errs[i + 1] <= errs[i] * (1 + 1e-12) for i in range(len(errs) - 1))
    # the explicit-operator CG and the GVT-operator CG agree
    xe, _, _, _ = O.cg(None, D, T, f, s, w.y, w.lam, w.iters, kernel=O.KRONECKER, explicit=True)
    assert rel(xe, x) < 1e-10


def test_cg_breakdown_on_indefinite_operator():
    """The p.Ap <= 0 exit (oracle.c O5) reached with lambda >= 0: an indefinite
    "Gram" D = diag(a, -1), T = [[1]], training pairs (0,0) and (1,0), so K = diag(a, -1) exactly.
    Arithmetic fixes where CG breaks down:
      y = (1, 1), a = 1:   p_1.Ap_1 = 1 - 1 = 0            -> breakdown at k = 1, x = 0;
      y = (1, 2), a = 1:   p_1.Ap_1 = 1 - 4 = -3           -> breakdown at k = 1, x = 0;
      y = (1, 1/2), a = 2: p_1.Ap_1 = 2 - 1/4 = 7/4 > 0, alpha = (5/4)/(7/4) = 5/7, x_1 = (5/7) y,
                           r_1 = y - (5/7) K y = (-3/7, 6/7), beta = (45/49)/(5/4) = 36/49,
                           p_2 = r_1 + beta y = (15/49, 60/49), p_2.Ap_2 = 2 (15/49)^2 - (60/49)^2 < 0
                           -> breakdown at k = 2 with the iterate x_1 returned, iters = 1.
    A negative lambda is a parameter error (OR_E_PARAM), not a breakdown."""
    kron = O.kernel_terms(O.KRONECKER)
    f, s = [0, 1], [0, 0]
    T = np.eye(1)
    for y in ([1.0, 1.0], [1.0, 2.0]):
        x, it, hist, rc = O.cg(kron, np.diag([1.0, -1.0]), T, f, s, y, 0.0, 5)
        assert rc == O.E_BREAKDOWN and it == 0 and np.all(x == 0), y
    x, it, hist, rc = O.cg(kron, np.diag([2.0, -1.0]), T, f, s, [1.0, 0.5], 0.0, 5)
    assert rc == O.E_BREAKDOWN and it == 1
    assert np.allclose(x, [5.0 / 7.0, 5.0 / 14.0], rtol=0, atol=1e-15)
    assert hist[1] == pytest.approx(np.hypot(3.0 / 7.0, 6.0 / 7.0) / np.hypot(1.0, 0.5), rel=1e-14)
    # the same system with a positive shift that makes it SPD (lambda = 2: diag(4, 1)) converges
    x, it, _, rc = O.cg(kron, np.diag([2.0, -1.0]), T, f, s, [1.0, 0.5], 2.0, 5)
    assert rc == O.OK and np.allclose(x, [0.25, 0.5], atol=1e-15)
    with pytest.raises(O.OracleError) as e:
        O.cg(kron, np.eye(2), T, f, s, [1.0, 0.0], -1.0, 3)
    assert e.value.code == O.E_PARAM


def test_cg_residual_mode_matches_scipy_cg():
    """Residual-mode stopping (reading S14: stop after iteration k when the recursive residual
    ||r_k|| / ||y|| <= tol) against scipy.sparse.linalg.cg(rtol=tol, x0=0) on C1's explicit system
    (K + lambda I): the same Hestenes-Stiefel recurrences with the same recursive residual test, so
    the iteration counts (SciPy's callback count) and the returned weights agree.  The 2I system
    stops after one iteration with an exactly zero residual."""
    from scipy.sparse.linalg import cg as scipy_cg
    w = synth.config1()
    D = O.gram(O.BASE_GAUSSIAN, w.Xd, gamma=w.gamma)
    T = O.gram(O.BASE_GAUSSIAN, w.Xt, gamma=w.gamma)
    f, s = w.train_first, w.train_second
    A = O.explicit_matrix(O.KRONECKER, D, T, f, s, f, s) + w.lam * np.eye(w.n)
    y = w.y.astype(np.float64)
    kron = O.kernel_terms(O.KRONECKER)
    lam_min = np.linalg.eigvalsh(A)[0]
    for tol in (1e-2, 1e-4, 1e-7):
        calls = []
        xs, info = scipy_cg(A, y, x0=np.zeros(w.n), rtol=tol, atol=0.0, maxiter=200, callback=calls.append)
        assert info == 0
        x, it, hist, rc = O.cg(kron, D, T, f, s, y, w.lam, 200, rel_tol=tol)
        assert rc == O.OK and it == len(calls), (tol, it, len(calls))
        assert hist[-1] <= tol < hist[-2]
        # the true residuals at exit are within the tolerance up to fp64 drift of the recursion,
        # and the two exits are within ||A^-1|| (||r|| + ||r_scipy||) of each other
        res, res_s = np.linalg.norm(y - A @ x), np.linalg.norm(y - A @ xs)
        assert res / np.linalg.norm(y) <= tol * (1 + 1e-6)
        assert np.linalg.norm(x - xs) <= (res + res_s) / lam_min * (1 + 1e-9)
    # 2I: one iteration, zero residual, a = y / 2
    fg, sg = np.repeat(np.arange(3), 2), np.tile(np.arange(2), 3)
    yg = np.array([1.0, -2.0, 0.5, 4.0, 3.0, -1.0])
    x, it, hist, rc = O.cg(kron, np.eye(3), np.eye(2), fg, sg, yg, 1.0, 10, rel_tol=1e-12)
    assert rc == O.OK and it == 1 and hist[-1] == 0.0 and np.allclose(x, yg / 2, atol=1e-15)


def test_predict_spec_example():
    """a=[1], train pair (0,0), Kronecker -> score(i,j) = D[i,0] T[j,0]."""
    rng = np.random.default_rng(2)
    Fd, Ft = rng.standard_normal((4, 2)), rng.standard_normal((3, 2))
    D, T = Fd @ Fd.T, Ft @ Ft.T
    of, os_ = np.repeat(np.arange(4), 3), np.tile(np.arange(3), 4)
    u = O.gvt_matvec(O.kernel_terms(O.KRONECKER), D, T, of, os_, [0], [0], [1.0])
    assert np.allclose(u, D[of, 0] * T[os_, 0], atol=1e-15)
    assert np.all(O.gvt_matvec(O.kernel_terms(O.KRONECKER), D, T, of, os_, [0], [0], [0.0]) == 0)


# ----------------------------------------------------------------------------- plumbing
@pytest.mark.parametrize("mode", [0, 1])
def test_sort_plan_matches_numpy_stable_sort(mode):
    rng = np.random.default_rng(8)
    m, q, n = 37, 23, 5000
    f, s = rng.integers(0, m, n), rng.integers(0, q, n)
    perm, rp = O.sort_plan(f, s, m, q, mode=mode)
    ref = np.argsort(f, kind="stable") if mode == 0 else np.lexsort((np.arange(n), s, f))
    assert np.array_equal(perm, ref)
    assert np.array_equal(rp, np.searchsorted(np.sort(f), np.arange(m + 1), side="left"))


# ----------------------------------------------------------------------------- MINRES (O5b)
def _explicit_system(w, kernel=O.KRONECKER):
    D = O.gram(w.base, w.Xd, gamma=w.gamma)
    T = None if w.Xt is None else O.gram(w.base, w.Xt, gamma=w.gamma)
    K = O.explicit_matrix(kernel, D, T, w.train_first, w.train_second, w.train_first, w.train_second)
    return D, T, K


def test_minres_scalar_systems():
    """SPEC.md minres_solve examples: 2I -> y/2 in one iteration; y = 0 -> 0 after 0
    iterations; K = I with lambda = 0 -> a = y; the single-pair ridge (1 + 1) a = 2."""
    f, s = np.repeat(np.arange(3), 2), np.tile(np.arange(2), 3)
    y = np.array([1.0, -2.0, 0.5, 4.0, 3.0, -1.0])
    kron = O.kernel_terms(O.KRONECKER)
    x, it, hist, rc = O.minres(kron, np.eye(3), np.eye(2), f, s, y, 1.0, 5)
    assert rc == O.OK and it == 1 and np.allclose(x, y / 2, atol=1e-15) and hist[-1] <= 1e-15
    x, it, hist, rc = O.minres(kron, np.eye(3), np.eye(2), f, s, np.zeros(6), 1.0, 5)
    assert it == 0 and np.all(x == 0)
    x, it, _, _ = O.minres(kron, np.eye(3), np.eye(2), f, s, y, 0.0, 5)
    assert np.allclose(x, y, atol=1e-15)
    r = SPEC["ridge_single_pair"]
    x, it, _, rc = O.minres(kron, [[r["D"]]], [[r["T"]]], [0], [0], [r["y"]], r["lambda"], 3)
    assert x[0] == pytest.approx(r["a"], abs=1e-15)


def test_minres_iterates_match_scipy_minres():
    """The paper ran scipy.sparse.linalg.minres: the oracle's iterates x_k equal
    SciPy's (same x0 = 0, no preconditioner) on the explicit C1 system up to rounding.  The two
    sum in different orders and Lanczos amplifies that (measured: 2e-15 at k = 1, 1e-9 at k = 12,
    2e-5 at k = 16, back to 1e-14 by k = 23, 1e-9 at k = 30 -- the same spread appears between
    the oracle's own explicit and GVT operators), so iterates are compared for k <= 12 at 1e-8
    and at k = 30 at 1e-7."""
    from scipy.sparse.linalg import minres as sp_minres
    w = synth.config1()
    D, T, K = _explicit_system(w)
    A = K + w.lam * np.eye(w.n)
    y = w.y.astype(np.float64)
    ref = []
    sp_minres(A, y, rtol=0.0, maxiter=30, callback=lambda xk: ref.append(xk.copy()))
    x, it, hist, rc, xh = O.minres(O.kernel_terms(O.KRONECKER), D, T, w.train_first, w.train_second, w.y, w.lam, 30,
                                   history=True)
    assert it == 30 and len(ref) == 30
    for k in range(1, 13):
        assert rel(xh[k], ref[k - 1]) < 1e-8, k
    assert rel(xh[30], ref[29]) < 1e-7


def test_minres_krylov_minimality_and_residual_estimate():
    """MINRES's defining property: x_k minimises ||y - A x|| over the Krylov space
    K_k(A, y) = span{y, Ay, ..., A^{k-1} y}.  Checked against numpy lstsq over an explicit
    orthonormal Krylov basis on a seeded 40-pair instance (all 9 kernels' K are symmetric);
    the recursive estimate phibar_k / ||y|| equals the true relative residual."""
    for kernel in (O.KRONECKER, O.SYMMETRIC, O.MLPK, O.POLY2D):
        hom = kernel in HOM
        w = synth.tiny(7, m=6, q=5, n=40, homogeneous=hom, duplicates=False)
        D, T, K = _explicit_system(w, kernel)
        A = K + 0.3 * np.eye(w.n)
        y = w.y.astype(np.float64)
        x, it, hist, rc, xh = O.minres(None, D, T, w.train_first, w.train_second, y, 0.3, 12, kernel=kernel,
                                       explicit=True, history=True)
        V = np.zeros((w.n, 0))
        b = y.copy()
        for k in range(1, it + 1):
            b = b / np.linalg.norm(b)
            v = b - V @ (V.T @ b)
            v -= V @ (V.T @ v)
            V = np.hstack([V, (v / np.linalg.norm(v))[:, None]])
            c, *_ = np.linalg.lstsq(A @ V, y, rcond=None)
            rmin = np.linalg.norm(y - A @ V @ c)
            rk = np.linalg.norm(y - A @ xh[k])
            assert rk == pytest.approx(rmin, rel=1e-7, abs=1e-12 * np.linalg.norm(y)), (kernel, k)
            assert hist[k] == pytest.approx(rk / np.linalg.norm(y), rel=1e-7, abs=1e-13), (kernel, k)
            b = A @ b


def test_minres_converges_monotone_on_C1_and_large_lambda_limit():
    """On C1 the relative residual history is non-increasing (SPEC.md: 'residual_history is
    non-increasing', 1e-12 slack) and 50 iterations reach the dense direct solve; with
    lambda = 1e6, a -> y / lambda (SPEC regularization limit, 1e-3)."""
    w = synth.config1()
    D, T, K = _explicit_system(w)
    kron = O.kernel_terms(O.KRONECKER)
    x, it, hist, rc = O.minres(kron, D, T, w.train_first, w.train_second, w.y, w.lam, 50)
    assert rc == O.OK and it == 50
    assert all(hist[k + 1] <= hist[k] * (1 + 1e-12) for k in range(len(hist) - 1))
    xs = np.linalg.solve(K + w.lam * np.eye(w.n), w.y.astype(np.float64))
    assert rel(x, xs) < 1e-10
    x, _, _, _ = O.minres(kron, D, T, w.train_first, w.train_second, w.y, 1e6, 10)
    assert rel(x, w.y / 1e6) < 1e-3


# ----------------------------------------------------------------------------- AUC (O8) and early stopping
def test_auc_matches_sklearn_with_ties():
    """AUC by definition equals sklearn.metrics.roc_auc_score (a library routine) on seeded
    inputs with heavy ties, for 0/1 and -1/+1 labels."""
    from sklearn.metrics import roc_auc_score
    rng = np.random.default_rng(5)
    for trial in range(20):
        n = int(rng.integers(2, 300))
        lab = rng.integers(0, 2, n)
        lab[0], lab[-1] = 0, 1
        sc = np.round(rng.standard_normal(n), 1) if trial % 2 else rng.standard_normal(n)
        assert O.auc(lab, sc) == pytest.approx(roc_auc_score(lab, sc), abs=1e-15)
        assert O.auc(2 * lab - 1, sc) == pytest.approx(roc_auc_score(lab, sc), abs=1e-15)


def test_auc_invariants_and_errors():
    """SPEC.md invariants: invariant under a strictly increasing transform; auc(s) + auc(-s) = 1
    without ties; all-tied scores give 1/2; a single-class label set is an error."""
    rng = np.random.default_rng(6)
    lab = rng.integers(0, 2, 200)
    sc = rng.standard_normal(200)
    a = O.auc(lab, sc)
    assert O.auc(lab, np.exp(3 * sc) + 7) == a
    assert a + O.auc(lab, -sc) == pytest.approx(1.0, abs=1e-15)
    assert O.auc(lab, np.zeros(200)) == 0.5
    assert O.auc([1, 0], [0.2, 0.1]) == 1.0 and O.auc([1, 0], [0.1, 0.2]) == 0.0
    with pytest.raises(O.OracleError):
        O.auc([1, 1, 1], [0.1, 0.2, 0.3])


def test_early_stop_rule_spec_examples():
    """SPEC.md fit_early_stopping examples: strictly increasing for 5 iterations then flat,
    patience 3 -> best 5 (stop at 8); constant from iteration 1, patience 2 -> best 1, stop at 3."""
    assert O.early_stop_rule([.5, .6, .7, .8, .9, .9, .9, .9, .9, .9], 3)[:4] == (5, .9, 8, True)
    assert O.early_stop_rule([.7] * 6, 2) == (1, .7, 3, True)
    assert O.early_stop_rule([.1, .2], 5) == (2, .2, 2, False)


def test_fit_early_stopping_chessboard():
    """SPEC.md: chessboard 12x12, Kronecker, lambda = 1e-5, patience 10 stops in far fewer
    iterations than n (observed <= n/4); the XOR is learnable by the Kronecker kernel (PAPER.md
    Figure 1 caption), so the best validation AUC is 1 and a_best's validation scores give it."""
    w, vlab = synth.parity_grid("chessboard", 12, 12, seed=0)
    D = O.gram(O.BASE_LINEAR, w.Xd)
    T = O.gram(O.BASE_LINEAR, w.Xt)
    kron = O.kernel_terms(O.KRONECKER)
    for solver in ("minres", "cg"):
        best, best_auc, iters, hist, a = O.fit_early_stopping(kron, D, T, w.train_first, w.train_second, w.y,
                                                              w.test_first, w.test_second, vlab, 1e-5, 10, w.n,
                                                              solver)
        assert iters <= w.n // 4, (solver, iters)
        assert best_auc == 1.0 and hist[best - 1] == 1.0
        sc = O.gvt_matvec(kron, D, T, w.test_first, w.test_second, w.train_first, w.train_second, a)
        assert O.auc(vlab, sc) == best_auc


# ----------------------------------------------------------------------------- novel objects (O9)
def test_gvt_rect_spec_examples():
    """SPEC.md gvt_matvec / gvt_cost / gvt_op_count examples on the rectangular GvtProblem."""
    u, v, ops = O.gvt_rect([[2.0]], [[3.0]], [0], [0], [0], [0], [1.0])
    assert u[0] == 6.0 and v == 1 and ops == 2
    f, s = [0, 0, 1, 1], [0, 1, 0, 1]
    vec = np.array([0.3, -1.2, 2.5, 0.7])
    for var in (1, 2):
        u, _, _ = O.gvt_rect(np.eye(2), np.eye(2), f, s, f, s, vec, var)
        assert np.array_equal(u, vec)
    # (n_out=3, m_out=2, q_out=2, n_in=4, m_in=3, q_in=2): cost1 = 17, cost2 = 14
    rng = np.random.default_rng(1)
    A, B = rng.uniform(size=(2, 3)), rng.uniform(size=(2, 2))
    of, os_ = [0, 1, 1], [1, 0, 1]
    inf, ins = [0, 2, 1, 2], [1, 1, 0, 0]
    a = rng.standard_normal(4)
    u0, v0, ops0 = O.gvt_rect(A, B, of, os_, inf, ins, a, 0)
    u1, v1, ops1 = O.gvt_rect(A, B, of, os_, inf, ins, a, 1)
    assert (v0, ops0, v1, ops1) == (2, 14, 1, 17)
    assert rel(u0, u1) < 1e-14


def test_gvt_rect_equals_brute_force():
    """200 seeded rectangular instances (m_out != m_in, q_out != q_in, duplicates): both variants
    and auto equal the brute-force sum u_i = sum_j A[of_i, if_j] B[os_i, is_j] a_j (numpy fancy
    indexing) within 1e-12."""
    for seed in range(200):
        rng = np.random.default_rng(500 + seed)
        mo, mi, qo, qi = rng.integers(1, 8, 4)
        no, ni = rng.integers(0, 20, 2)
        A, B = rng.standard_normal((mo, mi)), rng.standard_normal((qo, qi))
        of, os_ = rng.integers(0, mo, no), rng.integers(0, qo, no)
        inf, ins = rng.integers(0, mi, ni), rng.integers(0, qi, ni)
        a = rng.standard_normal(ni)
        ref = (A[of][:, inf] * B[os_][:, ins]) @ a if no and ni else np.zeros(no)
        for var in (0, 1, 2):
            u, _, _ = O.gvt_rect(A, B, of, os_, inf, ins, a, var)
            assert rel(u, ref) < 1e-12, (seed, var)


def test_gvt_rect_roth_vec_trick():
    """Complete out and in grids: u = vec(A V B^T) (Roth's column lemma) with
    rectangular A (5 x 7) and B (4 x 3), checked against numpy matmul."""
    rng = np.random.default_rng(3)
    A, B = rng.standard_normal((5, 7)), rng.standard_normal((4, 3))
    V = rng.standard_normal((7, 3))
    inf, ins = np.repeat(np.arange(7), 3), np.tile(np.arange(3), 7)
    of, os_ = np.repeat(np.arange(5), 4), np.tile(np.arange(4), 5)
    for var in (1, 2):
        u, _, _ = O.gvt_rect(A, B, of, os_, inf, ins, V.reshape(-1), var)
        assert rel(u, (A @ V @ B.T).reshape(-1)) < 1e-13


@pytest.mark.parametrize("kernel", [k for k in K_ALL if k != O.CARTESIAN])
def test_explicit_rect_equals_union_gram_subblock(kernel):
    """Novel objects as a sub-block: with the training objects and the test objects stacked into
    one table, the cross-Gram is a sub-block of the union Gram, so the rectangular definition
    must equal the (pinned) square definition over global ids -- for every kernel but Cartesian
    (which the rectangular form rejects, reading N1)."""
    hom = kernel in HOM
    rng = np.random.default_rng(40 + kernel)
    Xd_tr, Xd_te = rng.standard_normal((6, 3)), rng.standard_normal((4, 3))
    Xt_tr, Xt_te = rng.standard_normal((5, 3)), rng.standard_normal((3, 3))
    Du = O.gram(O.BASE_GAUSSIAN, np.vstack([Xd_tr, Xd_te]), gamma=0.4)
    Tu = None if hom else O.gram(O.BASE_GAUSSIAN, np.vstack([Xt_tr, Xt_te]), gamma=0.4)
    mi, mo = 6, 4
    qi, qo = (6, 4) if hom else (5, 3)
    Dx = Du[mi:, :mi]
    Tx = None if hom else Tu[qi:, :qi]
    n_in, n_out = 30, 17
    inf, ins = rng.integers(0, mi, n_in), rng.integers(0, qi, n_in)
    of, os_ = rng.integers(0, mo, n_out), rng.integers(0, qo, n_out)
    a = rng.standard_normal(n_in)
    u = O.explicit_rect_matvec(kernel, Dx, Tx, of, os_, inf, ins, a)
    ref = O.explicit_matvec(kernel, Du, Tu, of + mi, os_ + qi, inf, ins, a)
    assert rel(u, ref) < 1e-13
    with pytest.raises(O.OracleError) as e:
        O.explicit_rect_matvec(O.CARTESIAN, Dx, Tu[qi:, :qi] if Tu is not None else np.ones((qo, qi)), of, os_,
                               inf, ins, a)
    assert e.value.code == O.E_KERNEL


# ----------------------------------------------------------------------------- Tanimoto (NEXT-4)
def test_tanimoto_spec_worked_values():
    """[1,1,0] vs [1,0,1] -> 1/3; identical nonzero -> 1; both all-zero -> 1 (T1)."""
    for case in SPEC["tanimoto_base"]["cases"]:
        k = O.gram(O.BASE_TANIMOTO, [case["v"]], [case["w"]])[0, 0]
        assert k == case["k"][0] / case["k"][1]


def test_tanimoto_equals_scipy_jaccard_and_is_psd():
    """Tanimoto on binary vectors = 1 - Jaccard distance (scipy cdist 'jaccard', a library
    routine; scipy defines 0/0 as distance 0, matching T1); the Gram is PSD; an entry other than
    0/1 is an error."""
    rng = np.random.default_rng(8)
    X = (rng.uniform(size=(60, 300)) < rng.uniform(0.01, 0.3, size=(60, 1))).astype(float)
    Y = (rng.uniform(size=(45, 300)) < 0.05).astype(float)
    X[3] = 0.0
    Y[7] = 0.0
    K = O.gram(O.BASE_TANIMOTO, X, Y)
    assert np.allclose(K, 1.0 - cdist(X.astype(bool), Y.astype(bool), "jaccard"), atol=1e-15, rtol=0)
    assert K[3, 7] == 1.0
    G = O.gram(O.BASE_TANIMOTO, X)
    assert np.all(np.diag(G) == 1.0)
    assert np.linalg.eigvalsh(G).min() >= -1e-10 * np.abs(G).max()
    with pytest.raises(O.OracleError):
        O.gram(O.BASE_TANIMOTO, [[0.0, 0.5]])


# ----------------------------------------------------------------------------- O7b compact relabel
def test_relabel_spec_worked_values():
    """SPEC.md:55-57 examples (golden file)."""
    for case in SPEC["relabel_compact"]["cases"]:
        bound = max(case["ids"]) + 1 if case["ids"] else 1
        compact, unique, count = O.relabel(case["ids"], bound)
        assert compact.tolist() == case["compact"]
        assert unique.tolist() == case["unique"]
        assert count == case["count"]


def test_relabel_matches_numpy_first_occurrence_and_invariants():
    """unique ids in first-occurrence order = numpy.unique's first indices sorted; compact ids
    reproduce the input through unique; idempotent on compact input;
    out-of-range ids are an index error."""
    rng = np.random.default_rng(17)
    for trial in range(40):
        bound = int(rng.integers(1, 300))
        n = int(rng.integers(0, 2000))
        ids = rng.integers(0, bound, n).astype(np.int32)
        compact, unique, count = O.relabel(ids, bound)
        vals, first = np.unique(ids, return_index=True)
        order = np.argsort(first, kind="stable")
        assert count == len(vals)
        assert np.array_equal(unique, vals[order])
        assert np.array_equal(unique[compact], ids)
        assert compact.size == 0 or (compact.min() >= 0 and compact.max() < count)
        c2, u2, k2 = O.relabel(compact, max(count, 1))
        assert k2 == count and np.array_equal(c2, compact) and np.array_equal(u2, np.arange(count))
    # brute force on tiny inputs: a dict in index order
    for trial in range(200):
        ids = rng.integers(0, 6, int(rng.integers(0, 9))).astype(np.int32)
        seen = {}
        for v in ids.tolist():
            seen.setdefault(v, len(seen))
        compact, unique, count = O.relabel(ids, 6)
        assert compact.tolist() == [seen[v] for v in ids.tolist()] and unique.tolist() == list(seen)
    with pytest.raises(Exception):
        O.relabel(np.array([0, 3], np.int32), 3)
