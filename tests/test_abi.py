"""C-ABI library checks that need no GPU (-m "not gpu"): libgvt.so loads, exports every
symbol include/gvt.h declares, host-only entry points behave, and error conventions."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2009_01054_b200 as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "gvt.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:gvt_status|const char \*)\s*(\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for must in ("gvt_matvec", "pairwise_krr_fit", "pairwise_predict", "gvt_gram", "gvt_kernel_terms",
                 "gvt_create", "gvt_destroy", "gvt_last_error", "gvt_comm_init", "gvt_sort_plan"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(G.library_path())
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(declared_functions()) <= set(G.EXPORTED)


def test_library_is_sm100a_fatbin():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", G.library_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_kernel_terms_match_oracle_decomposition():
    """The library's Corollary lists and the oracle's are written independently; they must agree."""
    for k in range(9):
        lib_terms = [t.as_tuple() for t in G.gvt_kernel_terms(k)]
        ora_terms = [t.as_tuple() for t in O.kernel_terms(k)]
        assert lib_terms == ora_terms, k
    with pytest.raises(G.GvtError) as e:
        G.gvt_kernel_terms(99)
    assert e.value.code == G.E_KERNEL


def test_partition_balanced_contiguous():
    rng = np.random.default_rng(0)
    deg = rng.integers(1, 1000, 5000)
    for world in (1, 2, 3, 4, 8):
        b = G.gvt_partition(deg, world)
        assert b[0] == 0 and b[-1] == len(deg) and np.all(np.diff(b) >= 0)
        loads = np.array([deg[b[g]:b[g + 1]].sum() for g in range(world)])
        assert loads.sum() == deg.sum()
        assert loads.max() - loads.min() <= 2 * deg.max()
    assert list(G.gvt_partition([], 2)) == [0, 0, 0]
    with pytest.raises(G.GvtError):
        G.gvt_partition([1, -1], 2)


def test_null_context_is_an_error_not_a_crash():
    lib = ctypes.CDLL(G.library_path())
    lib.gvt_set_option.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_double]
    assert lib.gvt_set_option(None, 0, 1.0) == G.E_STATE


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(G.GvtError) as e:
        G.Context(0)
    assert e.value.code in (G.E_CUDA, G.E_PARAM)
