"""fp64 CPU oracle for the GVT hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2009_01054_b200``) never imports it and shares no code with it; the only
module both sides use is ``synth`` (seeded inputs, no method arithmetic).

Thin ctypes wrapper around ``oracle/liboracle.so`` (built from ``oracle.c`` by
``build()``; plain C, -O2 -ffp-contract=off, OpenMP).  Every function converts its
inputs to float64 and returns float64.  See oracle.c for the paper passage each
function follows and DESIGN.md for the readings and the pins.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# enums (oracle-side copies; the CUDA side has its own in include/gvt.h)
LINEAR, POLY2D, GAUSSIAN, KRONECKER, SYMMETRIC, ANTISYMMETRIC, RANKING, MLPK, CARTESIAN = range(9)
HOMOGENEOUS = (SYMMETRIC, ANTISYMMETRIC, RANKING, MLPK)
BASE_LINEAR, BASE_GAUSSIAN, BASE_POLY, BASE_TANIMOTO = range(4)
DRUG, TARGET, ONES, IDENTITY = range(4)
FIRST, SECOND = 0, 1
OK, E_DIM, E_INDEX, E_HOMOGENEOUS, E_KERNEL, E_PARAM, E_BREAKDOWN, E_OOM = range(8)


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"oracle {what} failed with code {code}")
        self.code = code


class Term(ctypes.Structure):
    _fields_ = [("coef", ctypes.c_double), ("left", ctypes.c_int32), ("right", ctypes.c_int32),
                ("row_sel_left", ctypes.c_int32), ("row_sel_right", ctypes.c_int32),
                ("col_sel_left", ctypes.c_int32), ("col_sel_right", ctypes.c_int32)]

    def as_tuple(self):
        return (self.coef, self.left, self.right, self.row_sel_left, self.row_sel_right,
                self.col_sel_left, self.col_sel_right)


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no BLAS, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
               "-std=c11", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.oracle_gram.argtypes = [i32, P, i64, P, i64, i64, dbl, dbl, i32, P]
        L.oracle_kernel_value.argtypes = [i32, P, i64, P, i64, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32, ctypes.c_int32]
        L.oracle_kernel_value.restype = dbl
        L.oracle_explicit_matrix.argtypes = [i32, P, i64, P, i64, P, P, i64, P, P, i64, P]
        L.oracle_explicit_matvec.argtypes = [i32, P, i64, P, i64, P, P, i64, P, P, i64, P, P]
        L.oracle_kernel_terms.argtypes = [i32, P, P]
        L.oracle_term_gvt.argtypes = [P, P, i64, P, i64, P, P, i64, P, P, i64, P, i32, P, P]
        L.oracle_term_cost.argtypes = [P, i64, i64, i32, P, P, i64, P, P, i64, P, P]
        L.oracle_gvt_matvec.argtypes = [P, i32, P, i64, P, i64, P, P, i64, P, P, i64, P, i32, P, P]
        L.oracle_cg.argtypes = [i32, P, i32, i32, P, i64, P, i64, P, P, i64, P, dbl, i32, dbl, P, P, P, P]
        L.oracle_minres.argtypes = [i32, P, i32, i32, P, i64, P, i64, P, P, i64, P, dbl, i32, dbl, P, P, P, P]
        L.oracle_auc.argtypes = [P, P, i64, P]
        L.oracle_explicit_rect_matvec.argtypes = [i32, P, i64, i64, P, i64, i64, P, P, i64, P, P, i64, P, P]
        L.oracle_gvt_rect.argtypes = [P, i64, i64, P, i64, i64, P, P, i64, P, P, i64, P, i32, P, P, P]
        L.oracle_sort_plan.argtypes = [P, P, i64, i64, i64, i32, P, P]
        L.oracle_relabel.argtypes = [P, i64, i64, P, P, P]
        L.oracle_num_threads.restype = i32
        L.oracle_set_num_threads.argtypes = [i32]
        _lib = L
    return _lib


def _d(a):
    return None if a is None else np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _check(rc, what):
    if rc != OK:
        raise OracleError(rc, what)


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP thread count for the timing legs (results do not depend on it)."""
    lib().oracle_set_num_threads(int(n))


def gram(base, X, Y=None, gamma=1.0, coef0=1.0, degree=2):
    """K[i,j] = k(X_i, Y_j) in fp64."""
    X = _d(X)
    Y = X if Y is None else _d(Y)
    K = np.empty((X.shape[0], Y.shape[0]), dtype=np.float64)
    _check(lib().oracle_gram(base, _p(X), X.shape[0], _p(Y), Y.shape[0], X.shape[1], gamma, coef0,
                             degree, _p(K)), "gram")
    return K


def kernel_value(kernel, D, T, out_pair, in_pair):
    D = _d(D)
    T = _d(T)
    return float(lib().oracle_kernel_value(kernel, _p(D), D.shape[0], _p(T), 0 if T is None else T.shape[0],
                                           int(out_pair[0]), int(out_pair[1]), int(in_pair[0]), int(in_pair[1])))


def explicit_matrix(kernel, D, T, of, os_, inf, ins):
    D, T = _d(D), _d(T)
    of, os_, inf, ins = _i(of), _i(os_), _i(inf), _i(ins)
    K = np.empty((len(of), len(inf)), dtype=np.float64)
    _check(lib().oracle_explicit_matrix(kernel, _p(D), D.shape[0], _p(T), 0 if T is None else T.shape[0],
                                        _p(of), _p(os_), len(of), _p(inf), _p(ins), len(inf), _p(K)),
           "explicit_matrix")
    return K


def explicit_matvec(kernel, D, T, of, os_, inf, ins, a):
    D, T, a = _d(D), _d(T), _d(a)
    of, os_, inf, ins = _i(of), _i(os_), _i(inf), _i(ins)
    u = np.empty(len(of), dtype=np.float64)
    _check(lib().oracle_explicit_matvec(kernel, _p(D), D.shape[0], _p(T), 0 if T is None else T.shape[0],
                                        _p(of), _p(os_), len(of), _p(inf), _p(ins), len(inf), _p(a), _p(u)),
           "explicit_matvec")
    return u


def kernel_terms(kernel):
    arr = (Term * 16)()
    n = ctypes.c_int(0)
    _check(lib().oracle_kernel_terms(kernel, ctypes.cast(arr, ctypes.c_void_p), ctypes.byref(n)), "kernel_terms")
    return [arr[i] for i in range(n.value)]


def terms_array(terms):
    arr = (Term * max(1, len(terms)))()
    for i, t in enumerate(terms):
        if isinstance(t, Term):
            arr[i] = t
        else:
            arr[i] = Term(*t)
    return arr


def term_cost(term, m, q, homogeneous, of, os_, inf, ins):
    of, os_, inf, ins = _i(of), _i(os_), _i(inf), _i(ins)
    c1, c2 = ctypes.c_int64(), ctypes.c_int64()
    t = terms_array([term])
    _check(lib().oracle_term_cost(ctypes.cast(t, ctypes.c_void_p), m, q, int(homogeneous), _p(of), _p(os_), len(of),
                                  _p(inf), _p(ins), len(inf), ctypes.byref(c1), ctypes.byref(c2)), "term_cost")
    return c1.value, c2.value


def term_gvt(term, D, T, of, os_, inf, ins, a, variant=1):
    D, T, a = _d(D), _d(T), _d(a)
    of, os_, inf, ins = _i(of), _i(os_), _i(inf), _i(ins)
    u = np.zeros(len(of), dtype=np.float64)
    ops = ctypes.c_int64(0)
    t = terms_array([term])
    _check(lib().oracle_term_gvt(ctypes.cast(t, ctypes.c_void_p), _p(D), D.shape[0], _p(T),
                                 0 if T is None else T.shape[0], _p(of), _p(os_), len(of), _p(inf), _p(ins),
                                 len(inf), _p(a), variant, _p(u), ctypes.byref(ops)), "term_gvt")
    return u, ops.value


def gvt_matvec(terms, D, T, of, os_, inf, ins, a, variant=1, return_ops=False):
    """u = sum over terms of the per-term GVT (O4), list order, variant 1/2/0=auto."""
    D, T, a = _d(D), _d(T), _d(a)
    of, os_, inf, ins = _i(of), _i(os_), _i(inf), _i(ins)
    u = np.zeros(len(of), dtype=np.float64)
    ops = ctypes.c_int64(0)
    t = terms_array(terms)
    _check(lib().oracle_gvt_matvec(ctypes.cast(t, ctypes.c_void_p), len(terms), _p(D), D.shape[0], _p(T),
                                   0 if T is None else T.shape[0], _p(of), _p(os_), len(of), _p(inf), _p(ins),
                                   len(inf), _p(a), variant, _p(u), ctypes.byref(ops)), "gvt_matvec")
    return (u, ops.value) if return_ops else u


def _solve(fn, name, terms, D, T, f, s, y, lam, max_iter, rel_tol, kernel, explicit, history):
    D, T, y = _d(D), _d(T), _d(y)
    f, s = _i(f), _i(s)
    n = len(f)
    x = np.zeros(n, dtype=np.float64)
    it = ctypes.c_int(0)
    hist = np.full(max_iter + 1, np.nan)
    xh = np.zeros((max_iter + 1, n), dtype=np.float64) if history else None
    tt = terms_array(terms if terms else [])
    rc = fn(kernel, ctypes.cast(tt, ctypes.c_void_p), len(terms) if terms else 0, int(explicit),
            _p(D), D.shape[0], _p(T), 0 if T is None else T.shape[0], _p(f), _p(s), n, _p(y),
            float(lam), int(max_iter), float(rel_tol), _p(x), ctypes.byref(it), _p(hist), _p(xh))
    if rc not in (OK, E_BREAKDOWN):
        raise OracleError(rc, name)
    out = (x, it.value, hist[: it.value + 1], rc)
    return out + (xh[: it.value + 1],) if history else out


def cg(terms, D, T, f, s, y, lam, max_iter, rel_tol=0.0, kernel=-1, explicit=False, history=False):
    """CG on (K + lam I) a = y (O5).  Returns (a, iters, relres_hist, code[, iterates])."""
    return _solve(lib().oracle_cg, "cg", terms, D, T, f, s, y, lam, max_iter, rel_tol, kernel, explicit, history)


def minres(terms, D, T, f, s, y, lam, max_iter, rel_tol=0.0, kernel=-1, explicit=False, history=False):
    """MINRES on (K + lam I) a = y (O5b).  Returns (a, iters, relres_hist, code[, iterates])."""
    return _solve(lib().oracle_minres, "minres", terms, D, T, f, s, y, lam, max_iter, rel_tol, kernel, explicit,
                  history)


def auc(labels, scores):
    """Mann-Whitney AUC by its definition (O8); positives are labels > 0."""
    lab, sc = _d(labels), _d(scores)
    out = ctypes.c_double(0.0)
    _check(lib().oracle_auc(_p(lab), _p(sc), len(lab), ctypes.byref(out)), "auc")
    return out.value


def early_stop_rule(auc_seq, patience):
    """The early-stopping rule of PAPER.md:852-856 ("until the AUC stops increasing in
    Z_validation for a given number of iterations") as SPEC.md fit_early_stopping states it:
    auc_seq[k-1] is the validation AUC after iteration k = 1, 2, ...; stop after `patience`
    consecutive iterations without STRICT improvement over the best so far; the best
    iteration is the earliest one reaching the maximum.  Returns (best_iter, best_auc,
    iters_used, stopped): iters_used = the iteration at which the rule fired (stopped=True)
    or len(auc_seq)."""
    best, best_it, bad = -np.inf, 0, 0
    for k, a in enumerate(auc_seq, start=1):
        if a > best:
            best, best_it, bad = a, k, 0
        else:
            bad += 1
            if bad >= patience:
                return best_it, best, k, True
    return best_it, best, len(auc_seq), False


def fit_early_stopping(terms, D, T, f, s, y, vf, vs, vlab, lam, patience, max_iter, solver="minres"):
    """Early-stopping ridge regression (SPEC.md fit_early_stopping): run the
    solver on the inner sample; after every iteration k predict the validation pairs with the
    iterate x_k (O6: scores = K_val,inner x_k by the per-term GVT), take their AUC (O8) and
    apply early_stop_rule.  Returns (best_iter, best_auc, iters_run, auc_hist, a_best) with
    auc_hist[k-1] the AUC after iteration k."""
    fn = minres if solver == "minres" else cg
    x, it, hist, rc, xh = fn(terms, D, T, f, s, y, lam, max_iter, history=True)
    aucs = []
    for k in range(1, it + 1):
        aucs.append(auc(vlab, gvt_matvec(terms, D, T, vf, vs, f, s, xh[k])))
        if early_stop_rule(aucs, patience)[3]:
            break
    best_it, best_auc, _, _ = early_stop_rule(aucs, patience)
    a_best = xh[best_it] if best_it > 0 else np.zeros(len(f))
    return best_it, best_auc, len(aucs), np.array(aucs), a_best


def explicit_rect_matvec(kernel, Dx, Tx, of, os_, inf, ins, a):
    """u_i = sum_j k(out_i, in_j) a_j on rectangular cross-Grams (O9): Dx (m_out x m_in),
    Tx (q_out x q_in) or None (homogeneous); out ids index rows, in ids columns."""
    Dx, Tx, a = _d(Dx), _d(Tx), _d(a)
    of, os_, inf, ins = _i(of), _i(os_), _i(inf), _i(ins)
    u = np.empty(len(of), dtype=np.float64)
    qo, qi = (0, 0) if Tx is None else Tx.shape
    _check(lib().oracle_explicit_rect_matvec(kernel, _p(Dx), Dx.shape[0], Dx.shape[1], _p(Tx), qo, qi, _p(of),
                                             _p(os_), len(of), _p(inf), _p(ins), len(inf), _p(a), _p(u)),
           "explicit_rect_matvec")
    return u


def gvt_rect(A, B, of, os_, inf, ins, a, variant=0):
    """SPEC GvtProblem matvec with rectangular factors (O9): returns (u, variant_used, op_count)."""
    A, B, a = _d(A), _d(B), _d(a)
    of, os_, inf, ins = _i(of), _i(os_), _i(inf), _i(ins)
    u = np.zeros(len(of), dtype=np.float64)
    v, ops = ctypes.c_int(0), ctypes.c_int64(0)
    _check(lib().oracle_gvt_rect(_p(A), A.shape[0], A.shape[1], _p(B), B.shape[0], B.shape[1], _p(of), _p(os_),
                                 len(of), _p(inf), _p(ins), len(inf), _p(a), int(variant), _p(u), ctypes.byref(v),
                                 ctypes.byref(ops)), "gvt_rect")
    return u, v.value, ops.value


def relabel(ids, bound):
    """SPEC.md:49-57 relabel_compact over ids in [0, bound): (compact int32[n], unique int32[count],
    count) with unique in first-occurrence order (O7b)."""
    v = _i(ids)
    n = len(v)
    compact = np.empty(n, dtype=np.int32)
    unique = np.empty(max(1, min(n, bound)), dtype=np.int32)
    cnt = np.zeros(1, dtype=np.int64)
    _check(lib().oracle_relabel(_p(v), n, bound, _p(compact), _p(unique), _p(cnt)), "relabel")
    return compact, unique[:int(cnt[0])].copy(), int(cnt[0])


def sort_plan(first, second, m, q, mode=0):
    """Stable sort by first id (mode 0) or (first, second) (mode 1): (perm int32, row_ptr int64)."""
    f, s = _i(first), _i(second)
    perm = np.empty(len(f), dtype=np.int32)
    rp = np.empty(m + 1, dtype=np.int64)
    _check(lib().oracle_sort_plan(_p(f), _p(s), len(f), m, q, mode, _p(perm), _p(rp)), "sort_plan")
    return perm, rp
