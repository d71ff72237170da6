"""paper_2009_01054_b200 -- thin Python binding of libgvt.so (include/gvt.h).

The generalized vec trick (GVT) hot path of "Generalized vec trick for fast learning of
pairwise kernel models" (arXiv 2009.01054) on B200 (sm_100a): base-kernel Grams, the GVT
matvec for every Corollary kernel, CG kernel ridge regression and prediction.

This module only marshals arguments: it turns torch tensors (CUDA or CPU) and numpy
arrays into plain pointers and sizes and calls the C ABI of the same name.  Every step
of the computation runs in the library's CUDA kernels; there is no Python or CPU
fallback -- importing fails loudly if libgvt.so is missing, and every call raises
GvtError on a non-OK status (e.g. no CUDA device).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GVT_LIBRARY") or os.path.join(_HERE, "libgvt.so")  # override: A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libgvt.so not built at {LIB_PATH}: run `python -m paper_2009_01054_b200.build` "
                      "(the CUDA extension is required; there is no fallback)")

_lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)

# ---------------------------------------------------------------------------- enums (gvt.h)
OK, E_DIM, E_INDEX, E_HOMOGENEOUS, E_KERNEL, E_PARAM, E_BREAKDOWN, E_CUDA, E_NCCL, E_OOM, E_STATE = range(11)
LINEAR, POLY2D, GAUSSIAN, KRONECKER, SYMMETRIC, ANTISYMMETRIC, RANKING, MLPK, CARTESIAN = range(9)
BASE_LINEAR, BASE_GAUSSIAN, BASE_POLY, BASE_TANIMOTO = range(4)
FACTOR_DRUG, FACTOR_TARGET, FACTOR_ONES, FACTOR_IDENTITY = range(4)
SEL_FIRST, SEL_SECOND = 0, 1
OPT_ENGINE, OPT_DENSE_THRESHOLD, OPT_PROFILE, OPT_GRAM_ENGINE, OPT_TC_PRECISION = range(5)
PREC_FP16X3, PREC_TF32X3 = 0, 1
ENGINE_AUTO, ENGINE_SPARSE, ENGINE_DENSE, ENGINE_TINY, ENGINE_SMALL = 0, 1, 2, 3, 4
OPT_SLABS = 5
OPT_GEMM_CTA = 6
OPT_GRAPHS = 7
OPT_SOLVER = 8
OPT_EXCHANGE = 9
OPT_CG_VARIANT = 10
OPT_SORTED_FIT = 11
OPT_KBLOCK_SKIP = 12
OPT_STAGE2 = 13
OPT_COMPACT = 14
SOLVER_CG, SOLVER_MINRES = 0, 1
HOMOGENEOUS_KERNELS = (SYMMETRIC, ANTISYMMETRIC, RANKING, MLPK)
MAX_KINDS = 32


class GvtError(RuntimeError):
    def __init__(self, code: int, where: str):
        msg = _lib.gvt_last_error().decode(errors="replace")
        super().__init__(f"{where}: status {code}: {msg}")
        self.code = code


class Term(ctypes.Structure):
    """gvt_term: value = coef * L[row_sel_left(o), col_sel_left(i)] * R[row_sel_right(o), col_sel_right(i)]."""
    _fields_ = [("coef", ctypes.c_double), ("left", ctypes.c_int32), ("right", ctypes.c_int32),
                ("row_sel_left", ctypes.c_int32), ("row_sel_right", ctypes.c_int32),
                ("col_sel_left", ctypes.c_int32), ("col_sel_right", ctypes.c_int32)]

    def as_tuple(self):
        return (self.coef, self.left, self.right, self.row_sel_left, self.row_sel_right, self.col_sel_left,
                self.col_sel_right)


class Stats(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("n_kinds", ctypes.c_int32),
                ("names", (ctypes.c_char * 32) * MAX_KINDS), ("counts", ctypes.c_int64 * MAX_KINDS),
                ("ms", ctypes.c_double * MAX_KINDS), ("last_engine", ctypes.c_int32), ("world", ctypes.c_int32),
                ("last_exchange", ctypes.c_int32)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_lib.gvt_last_error.restype = ctypes.c_char_p
_lib.gvt_create.argtypes = [ctypes.POINTER(_P), ctypes.c_int, _P]
_lib.gvt_destroy.argtypes = [_P]
_lib.gvt_set_stream.argtypes = [_P, _P]
_lib.gvt_set_option.argtypes = [_P, ctypes.c_int, ctypes.c_double]
_lib.gvt_get_stats.argtypes = [_P, ctypes.POINTER(Stats)]
_lib.gvt_reset_stats.argtypes = [_P]
_lib.gvt_nccl_unique_id.argtypes = [_P]
_lib.gvt_comm_init.argtypes = [_P, _P, ctypes.c_int, ctypes.c_int]
_lib.gvt_partition.argtypes = [_P, _I64, ctypes.c_int, _P]
_lib.gvt_slab_bounds.argtypes = [_P, _I64, ctypes.c_int, _P]
_lib.gvt_kernel_terms.argtypes = [ctypes.c_int, _P, ctypes.POINTER(ctypes.c_int)]
_lib.gvt_gram.argtypes = [_P, ctypes.c_int, _P, _I64, _I64, ctypes.c_double, ctypes.c_double, ctypes.c_int, _P]
_lib.gvt_matvec.argtypes = [_P, _P, _I64, _P, _I64, _P, _P, _I64, _P, _P, _I64, _P, _P, ctypes.c_int, _P]
_lib.pairwise_krr_fit.argtypes = [_P, _P, _I64, _P, _I64, _P, _P, _I64, _P, _P, ctypes.c_int, ctypes.c_double,
                                  ctypes.c_int, ctypes.c_double, _P, ctypes.POINTER(ctypes.c_int), _P]
_lib.pairwise_predict.argtypes = [_P, _P, _I64, _P, _I64, _P, _P, _I64, _P, _P, _I64, _P, _P, ctypes.c_int, _P]
_lib.gvt_sort_plan.argtypes = [_P, _P, _P, _I64, _I64, _I64, ctypes.c_int, _P, _P]
_lib.gvt_relabel_compact.argtypes = [_P, _P, _I64, _I64, _P, _P, _P]
_lib.pairwise_krr_fit_early_stopping.argtypes = [_P, _P, _I64, _P, _I64, _P, _P, _I64, _P, _P, _P, _I64, _P, _P,
                                                 ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int, _P,
                                                 ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double),
                                                 ctypes.POINTER(ctypes.c_int), _P]
_lib.gvt_auc.argtypes = [_P, _P, _P, _I64, ctypes.POINTER(ctypes.c_double)]
HOST_ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t)
_lib.gvt_comm_init_host.argtypes = [_P, ctypes.c_int, ctypes.c_int, HOST_ALLGATHER_FN, _P]
_lib.gvt_gram_cross.argtypes = [_P, ctypes.c_int, _P, _I64, _P, _I64, _I64, ctypes.c_double, ctypes.c_double,
                                ctypes.c_int, _P]
_lib.gvt_matvec_rect.argtypes = [_P, _P, _I64, _I64, _P, _I64, _I64, _P, _P, _I64, _P, _P, _I64, _P, _P, ctypes.c_int,
                                 ctypes.c_int, _P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64)]
_lib.pairwise_predict_rect.argtypes = [_P, _P, _I64, _I64, _P, _I64, _I64, _P, _P, _I64, _P, _P, _I64, _P, _P,
                                       ctypes.c_int, _P]

_lib.gvt_solver_direction.argtypes = [_P, _P, _I64]
_lib.gvt_slab_bounds_cost.argtypes = [_P, _I64, ctypes.c_int, ctypes.c_double, ctypes.c_double, _P]

EXPORTED = ["gvt_slab_bounds", "gvt_solver_direction", "gvt_slab_bounds_cost",
            "gvt_create", "gvt_destroy", "gvt_set_stream", "gvt_set_option", "gvt_get_stats", "gvt_reset_stats",
            "gvt_nccl_unique_id", "gvt_comm_init", "gvt_partition", "gvt_kernel_terms", "gvt_gram", "gvt_matvec",
            "pairwise_krr_fit", "pairwise_predict", "gvt_sort_plan", "gvt_last_error",
            "pairwise_krr_fit_early_stopping", "gvt_auc", "gvt_gram_cross", "gvt_matvec_rect",
            "pairwise_predict_rect", "gvt_comm_init_host", "gvt_relabel_compact"]


def _check(code: int, where: str):
    if code != OK:
        raise GvtError(code, where)


# ---------------------------------------------------------------------------- marshalling
def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _ptr(x, dtype: str, what: str):
    """Plain pointer of a contiguous array (torch tensor on any device, or numpy)."""
    if x is None:
        return None
    if _is_torch(x):
        import torch
        want = {"f32": torch.float32, "i32": torch.int32, "i64": torch.int64, "f64": torch.float64}[dtype]
        if x.dtype != want or not x.is_contiguous():
            raise TypeError(f"{what}: expected a contiguous {want} tensor, got {x.dtype}")
        return x.data_ptr() if x.numel() else None
    want = {"f32": np.float32, "i32": np.int32, "i64": np.int64, "f64": np.float64}[dtype]
    if not isinstance(x, np.ndarray) or x.dtype != want or not x.flags.c_contiguous:
        raise TypeError(f"{what}: expected a C-contiguous numpy {np.dtype(want).name} array")
    return x.ctypes.data if x.size else None


def _n(x):
    if x is None:
        return 0
    return int(x.numel()) if _is_torch(x) else int(x.size)


def _empty_like_input(ref, n, dtype="f32"):
    if _is_torch(ref):
        import torch
        return torch.empty(n, dtype={"f32": torch.float32, "i32": torch.int32, "i64": torch.int64}[dtype],
                           device=ref.device)
    return np.empty(n, dtype={"f32": np.float32, "i32": np.int32, "i64": np.int64}[dtype])


def terms_array(terms: Sequence):
    arr = (Term * max(1, len(terms)))()
    for i, t in enumerate(terms):
        arr[i] = t if isinstance(t, Term) else Term(*t)
    return arr


# ---------------------------------------------------------------------------- C-ABI mirrors
def gvt_kernel_terms(kernel: int):
    arr = (Term * 16)()
    n = ctypes.c_int(0)
    _check(_lib.gvt_kernel_terms(kernel, ctypes.cast(arr, _P), ctypes.byref(n)), "gvt_kernel_terms")
    return [arr[i] for i in range(n.value)]


def gvt_partition(deg, world: int):
    deg = np.ascontiguousarray(np.asarray(deg, dtype=np.int64))
    bounds = np.zeros(world + 1, dtype=np.int64)
    _check(_lib.gvt_partition(deg.ctypes.data if deg.size else None, deg.size, world, bounds.ctypes.data),
           "gvt_partition")
    return bounds


def gvt_slab_bounds(row_ptr, nslab: int):
    """Slab partition of pair-matrix rows used by the data-parallel path (host only)."""
    rp = np.ascontiguousarray(np.asarray(row_ptr, dtype=np.int64))
    bounds = np.zeros(nslab + 1, dtype=np.int64)
    _check(_lib.gvt_slab_bounds(rp.ctypes.data, rp.size - 1, nslab, bounds.ctypes.data), "gvt_slab_bounds")
    return bounds


def gvt_slab_bounds_cost(row_ptr, nslab: int, w_entry: float, w_row: float):
    """The engine's cost-balanced slab partition (host only)."""
    rp = np.ascontiguousarray(np.asarray(row_ptr, dtype=np.int64))
    bounds = np.zeros(nslab + 1, dtype=np.int64)
    _check(_lib.gvt_slab_bounds_cost(rp.ctypes.data, rp.size - 1, nslab, float(w_entry), float(w_row),
                                     bounds.ctypes.data), "gvt_slab_bounds_cost")
    return bounds


def gvt_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.gvt_nccl_unique_id(ctypes.cast(buf, _P)), "gvt_nccl_unique_id")
    return buf.raw


def gvt_last_error() -> str:
    return _lib.gvt_last_error().decode(errors="replace")


class Context:
    """Owns a gvt_ctx (gvt_create/gvt_destroy).  ``stream`` is a torch.cuda.Stream, a raw
    cudaStream_t integer, or None for torch's current stream on ``device`` (the legacy
    default stream if torch.cuda is unavailable)."""

    def __init__(self, device: int = 0, stream=None):
        self._h = _P()
        handle = self._stream_handle(device, stream)
        _check(_lib.gvt_create(ctypes.byref(self._h), device, handle), "gvt_create")
        self.device = device

    @staticmethod
    def _stream_handle(device, stream):
        if stream is None:
            try:
                import torch
                if torch.cuda.is_available():
                    return torch.cuda.current_stream(device).cuda_stream
            except Exception:
                pass
            return None
        if isinstance(stream, int):
            return stream
        return stream.cuda_stream

    def close(self):
        if self._h:
            _lib.gvt_destroy(self._h)
            self._h = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- options / stats
    def set_stream(self, stream):
        _check(_lib.gvt_set_stream(self._h, self._stream_handle(self.device, stream)), "gvt_set_stream")

    def set_option(self, opt: int, value: float):
        _check(_lib.gvt_set_option(self._h, opt, float(value)), "gvt_set_option")

    def stats(self) -> dict:
        s = Stats()
        _check(_lib.gvt_get_stats(self._h, ctypes.byref(s)), "gvt_get_stats")
        kinds = {}
        for k in range(s.n_kinds):
            name = bytes(s.names[k]).split(b"\0")[0].decode()
            if s.counts[k]:
                kinds[name] = {"count": int(s.counts[k]), "ms": float(s.ms[k])}
        return {"launches": int(s.launches), "kinds": kinds, "last_engine": int(s.last_engine), "world": int(s.world),
                "last_exchange": int(s.last_exchange)}

    def reset_stats(self):
        _check(_lib.gvt_reset_stats(self._h), "gvt_reset_stats")

    def comm_init(self, unique_id: bytes, rank: int, world: int):
        buf = ctypes.create_string_buffer(unique_id, 128)
        _check(_lib.gvt_comm_init(self._h, ctypes.cast(buf, _P), rank, world), "gvt_comm_init")

    def comm_init_host(self, rank: int, world: int, group=None):
        """gvt_comm_init_host with a torch.distributed (e.g. gloo) process group as the transport:
        every library collective becomes one all-gather of host bytes through `group`."""
        import torch
        import torch.distributed as dist

        def allgather(user, buf, nbytes):
            try:
                arr = np.ctypeslib.as_array(ctypes.cast(buf, ctypes.POINTER(ctypes.c_uint8)), shape=(world * nbytes,))
                mine = torch.from_numpy(arr[rank * nbytes:(rank + 1) * nbytes].copy())
                outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(outs, mine, group=group)
                for g in range(world):
                    arr[g * nbytes:(g + 1) * nbytes] = outs[g].numpy()
                return 0
            except Exception:  # pragma: no cover - surfaced as GVT_E_NCCL by the library
                return 1

        self._host_allgather = HOST_ALLGATHER_FN(allgather)  # keep the callback alive
        _check(_lib.gvt_comm_init_host(self._h, rank, world, self._host_allgather, None), "gvt_comm_init_host")

    # -- compute
    def gram(self, kind: int, X, gamma: float = 1.0, coef0: float = 1.0, degree: int = 2, out=None):
        m = int(X.shape[0])
        dim = int(X.shape[1]) if len(X.shape) > 1 else 0
        if out is None:
            out = _empty_like_input(X, m * m).reshape(m, m)
        _check(_lib.gvt_gram(self._h, kind, _ptr(X, "f32", "X"), m, dim, gamma, coef0, degree,
                             _ptr(out, "f32", "K")), "gvt_gram")
        return out

    def gram_cross(self, kind: int, X, Y, gamma: float = 1.0, coef0: float = 1.0, degree: int = 2, out=None):
        """gvt_gram_cross: K[i][j] = k(X_i, Y_j) (m x m2)."""
        m, m2 = int(X.shape[0]), int(Y.shape[0])
        dim = int(X.shape[1]) if len(X.shape) > 1 else 0
        if out is None:
            out = _empty_like_input(X, m * m2).reshape(m, m2)
        _check(_lib.gvt_gram_cross(self._h, kind, _ptr(X, "f32", "X"), m, _ptr(Y, "f32", "Y"), m2, dim, gamma, coef0,
                                   degree, _ptr(out, "f32", "K")), "gvt_gram_cross")
        return out

    def matvec_rect(self, Dx, Tx, out_first, out_second, in_first, in_second, a, terms, variant: int = 0, out=None):
        """gvt_matvec_rect on cross-Grams Dx (m_out x m_in), Tx (q_out x q_in) or None: returns
        (u, variant_used, op_count)."""
        m_out, m_in = int(Dx.shape[0]), int(Dx.shape[1])
        q_out, q_in = (0, 0) if Tx is None else (int(Tx.shape[0]), int(Tx.shape[1]))
        n_out, n_in = _n(out_first), _n(in_first)
        if out is None:
            out = _empty_like_input(a if a is not None else Dx, n_out)
        v, ops = ctypes.c_int(0), ctypes.c_int64(0)
        ta = terms_array(terms)
        _check(_lib.gvt_matvec_rect(self._h, _ptr(Dx, "f32", "Dx"), m_out, m_in, _ptr(Tx, "f32", "Tx"), q_out, q_in,
                                    _ptr(out_first, "i32", "out_first"), _ptr(out_second, "i32", "out_second"), n_out,
                                    _ptr(in_first, "i32", "in_first"), _ptr(in_second, "i32", "in_second"), n_in,
                                    _ptr(a, "f32", "a"), ctypes.cast(ta, _P), len(terms), int(variant),
                                    _ptr(out, "f32", "u"), ctypes.byref(v), ctypes.byref(ops)), "gvt_matvec_rect")
        return out, v.value, ops.value

    def predict_rect(self, Dx, Tx, test_first, test_second, train_first, train_second, a, terms, out=None):
        """pairwise_predict_rect: scores for novel objects (cross-Grams test x train)."""
        m_out, m_in = int(Dx.shape[0]), int(Dx.shape[1])
        q_out, q_in = (0, 0) if Tx is None else (int(Tx.shape[0]), int(Tx.shape[1]))
        n_test, n_train = _n(test_first), _n(train_first)
        if out is None:
            out = _empty_like_input(a if a is not None else Dx, n_test)
        ta = terms_array(terms)
        _check(_lib.pairwise_predict_rect(self._h, _ptr(Dx, "f32", "Dx"), m_out, m_in, _ptr(Tx, "f32", "Tx"), q_out,
                                          q_in, _ptr(test_first, "i32", "test_first"),
                                          _ptr(test_second, "i32", "test_second"), n_test,
                                          _ptr(train_first, "i32", "train_first"),
                                          _ptr(train_second, "i32", "train_second"), n_train, _ptr(a, "f32", "a"),
                                          ctypes.cast(ta, _P), len(terms), _ptr(out, "f32", "scores")),
               "pairwise_predict_rect")
        return out

    def matvec(self, D, T, out_first, out_second, in_first, in_second, a, terms, out=None):
        m = int(D.shape[0])
        q = int(T.shape[0]) if T is not None else 0
        n_out, n_in = _n(out_first), _n(in_first)
        if out is None:
            out = _empty_like_input(a if a is not None else D, n_out)
        ta = terms_array(terms)
        _check(_lib.gvt_matvec(self._h, _ptr(D, "f32", "D"), m, _ptr(T, "f32", "T"), q,
                               _ptr(out_first, "i32", "out_first"), _ptr(out_second, "i32", "out_second"), n_out,
                               _ptr(in_first, "i32", "in_first"), _ptr(in_second, "i32", "in_second"), n_in,
                               _ptr(a, "f32", "a"), ctypes.cast(ta, _P), len(terms), _ptr(out, "f32", "u")),
               "gvt_matvec")
        return out

    def fit(self, D, T, first, second, y, terms, lam: float, max_iter: int, rel_tol: float = 0.0, out=None,
            want_history: bool = True, raise_on_breakdown: bool = True):
        m = int(D.shape[0])
        q = int(T.shape[0]) if T is not None else 0
        n = _n(first)
        if out is None:
            out = _empty_like_input(y if y is not None else D, n)
        iters = ctypes.c_int(0)
        hist = np.full(max_iter + 1, np.nan) if want_history else None
        ta = terms_array(terms)
        code = _lib.pairwise_krr_fit(self._h, _ptr(D, "f32", "D"), m, _ptr(T, "f32", "T"), q,
                                     _ptr(first, "i32", "first"), _ptr(second, "i32", "second"), n,
                                     _ptr(y, "f32", "y"), ctypes.cast(ta, _P), len(terms), float(lam), int(max_iter),
                                     float(rel_tol), _ptr(out, "f32", "a_out"), ctypes.byref(iters),
                                     hist.ctypes.data if hist is not None else None)
        if code != OK and not (code == E_BREAKDOWN and not raise_on_breakdown):
            raise GvtError(code, "pairwise_krr_fit")
        h = hist[: iters.value + 1] if hist is not None else None
        return out, iters.value, h, code

    def solver_direction(self, n: int, like=None):
        """gvt_solver_direction: the last CG fit's next search direction p_{k+1} (caller order)."""
        out = _empty_like_input(like, n) if like is not None else np.empty(n, np.float32)
        _check(_lib.gvt_solver_direction(self._h, _ptr(out, "f32", "p_out"), n), "gvt_solver_direction")
        return out

    def fit_early_stopping(self, D, T, first, second, y, val_first, val_second, val_labels, terms, lam: float,
                           patience: int, max_iter: int, out=None):
        """pairwise_krr_fit_early_stopping: returns (a_best, best_iter, best_auc, iters_run, auc_hist)."""
        m = int(D.shape[0])
        q = int(T.shape[0]) if T is not None else 0
        n, n_val = _n(first), _n(val_first)
        if out is None:
            out = _empty_like_input(y if y is not None else D, n)
        best, iters = ctypes.c_int(0), ctypes.c_int(0)
        best_auc = ctypes.c_double(0.0)
        hist = np.full(max(1, max_iter), np.nan)
        ta = terms_array(terms)
        _check(_lib.pairwise_krr_fit_early_stopping(
            self._h, _ptr(D, "f32", "D"), m, _ptr(T, "f32", "T"), q, _ptr(first, "i32", "first"),
            _ptr(second, "i32", "second"), n, _ptr(y, "f32", "y"), _ptr(val_first, "i32", "val_first"),
            _ptr(val_second, "i32", "val_second"), n_val, _ptr(val_labels, "f32", "val_labels"), ctypes.cast(ta, _P),
            len(terms), float(lam), int(patience), int(max_iter), _ptr(out, "f32", "a_out"), ctypes.byref(best),
            ctypes.byref(best_auc), ctypes.byref(iters), hist.ctypes.data), "pairwise_krr_fit_early_stopping")
        return out, best.value, best_auc.value, iters.value, hist[: iters.value]

    def auc(self, labels, scores) -> float:
        """gvt_auc: Mann-Whitney AUC of scores against labels (positive iff label > 0)."""
        out = ctypes.c_double(0.0)
        _check(_lib.gvt_auc(self._h, _ptr(labels, "f32", "labels"), _ptr(scores, "f32", "scores"), _n(labels),
                            ctypes.byref(out)), "gvt_auc")
        return out.value

    def predict(self, D, T, test_first, test_second, train_first, train_second, a, terms, out=None):
        m = int(D.shape[0])
        q = int(T.shape[0]) if T is not None else 0
        n_test, n_train = _n(test_first), _n(train_first)
        if out is None:
            out = _empty_like_input(a if a is not None else D, n_test)
        ta = terms_array(terms)
        _check(_lib.pairwise_predict(self._h, _ptr(D, "f32", "D"), m, _ptr(T, "f32", "T"), q,
                                     _ptr(test_first, "i32", "test_first"), _ptr(test_second, "i32", "test_second"),
                                     n_test, _ptr(train_first, "i32", "train_first"),
                                     _ptr(train_second, "i32", "train_second"), n_train, _ptr(a, "f32", "a"),
                                     ctypes.cast(ta, _P), len(terms), _ptr(out, "f32", "scores")),
               "pairwise_predict")
        return out

    def relabel_compact(self, ids, bound: int):
        """(compact ids, unique ids in first-occurrence order, count)."""
        n = _n(ids)
        compact = _empty_like_input(ids, n, "i32")
        unique = _empty_like_input(ids, max(1, min(n, bound)), "i32")
        cnt = ctypes.c_int64(0)
        _check(_lib.gvt_relabel_compact(self._h, _ptr(ids, "i32", "ids"), n, bound, _ptr(compact, "i32", "compact"),
                                        _ptr(unique, "i32", "unique"), ctypes.byref(cnt)), "gvt_relabel_compact")
        return compact, unique[:cnt.value], cnt.value

    def sort_plan(self, first, second, m: int, q: int, mode: int = 0):
        n = _n(first)
        perm = _empty_like_input(first, n, "i32")
        rp = _empty_like_input(first, m + 1, "i64")
        _check(_lib.gvt_sort_plan(self._h, _ptr(first, "i32", "first"), _ptr(second, "i32", "second"), n, m, q, mode,
                                  _ptr(perm, "i32", "perm"), _ptr(rp, "i64", "row_ptr")), "gvt_sort_plan")
        return perm, rp


# module-level mirrors with the C names (argument marshalling only)
def gvt_create(device: int = 0, stream=None) -> Context:
    return Context(device, stream)


def gvt_destroy(ctx: Context):
    ctx.close()


def gvt_gram(ctx: Context, kind, X, gamma=1.0, coef0=1.0, degree=2, out=None):
    return ctx.gram(kind, X, gamma, coef0, degree, out)


def gvt_matvec(ctx: Context, D, T, out_first, out_second, in_first, in_second, a, terms, out=None):
    return ctx.matvec(D, T, out_first, out_second, in_first, in_second, a, terms, out)


def pairwise_krr_fit(ctx: Context, D, T, first, second, y, terms, lam, max_iter, rel_tol=0.0, out=None):
    return ctx.fit(D, T, first, second, y, terms, lam, max_iter, rel_tol, out)


def pairwise_predict(ctx: Context, D, T, test_first, test_second, train_first, train_second, a, terms, out=None):
    return ctx.predict(D, T, test_first, test_second, train_first, train_second, a, terms, out)


def pairwise_krr_fit_early_stopping(ctx: Context, D, T, first, second, y, val_first, val_second, val_labels, terms,
                                    lam, patience, max_iter, out=None):
    return ctx.fit_early_stopping(D, T, first, second, y, val_first, val_second, val_labels, terms, lam, patience,
                                  max_iter, out)


def gvt_auc(ctx: Context, labels, scores):
    return ctx.auc(labels, scores)


def gvt_gram_cross(ctx: Context, kind, X, Y, gamma=1.0, coef0=1.0, degree=2, out=None):
    return ctx.gram_cross(kind, X, Y, gamma, coef0, degree, out)


def gvt_matvec_rect(ctx: Context, Dx, Tx, out_first, out_second, in_first, in_second, a, terms, variant=0, out=None):
    return ctx.matvec_rect(Dx, Tx, out_first, out_second, in_first, in_second, a, terms, variant, out)


def pairwise_predict_rect(ctx: Context, Dx, Tx, test_first, test_second, train_first, train_second, a, terms,
                          out=None):
    return ctx.predict_rect(Dx, Tx, test_first, test_second, train_first, train_second, a, terms, out)


def gvt_relabel_compact(ctx: Context, ids, bound):
    return ctx.relabel_compact(ids, bound)


def gvt_solver_direction(ctx: Context, n, like=None):
    return ctx.solver_direction(n, like)


def gvt_sort_plan(ctx: Context, first, second, m, q, mode=0):
    return ctx.sort_plan(first, second, m, q, mode)


def library_path() -> str:
    return LIB_PATH
