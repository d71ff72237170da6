"""Symmetric upper-triangle GEMV (square Grams >= 6144 objects, sparse.cu k_symv_panel + k_symv_finish)
against the oracle (-m gpu).  The cheap Ranking form reduces the whole matvec to one GEMV with the Gram
(reading R1: the Gram is symmetric by definition), so a Ranking matvec on a homogeneous
domain of n >= 6144 objects runs the panel kernels; n = 6150 and 7003 are ragged (not multiples of
the 4-float quad, the 64-row chunk or the 1024-column panel: the library pads the Gram copy with
zeros), n = 8000 is C4's union domain size."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle as O
import paper_2009_01054_b200 as G
import synth


def rel(x, ref):
    x, ref = np.asarray(x, np.float64), np.asarray(ref, np.float64)
    return float(np.linalg.norm(x - ref) / np.linalg.norm(ref))


@pytest.fixture(scope="module")
def ctx():
    c = G.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("n_obj", [6150, 7003, 8000])
def test_ranking_symv_vs_oracle(ctx, n_obj):
    rng = np.random.default_rng(n_obj)
    X = rng.standard_normal((n_obj, 16)).astype(np.float32)
    D = np.ascontiguousarray(O.gram(G.BASE_GAUSSIAN, X, gamma=1 / 16), dtype=np.float32)
    n_in, n_out = 40000, 5000
    inf, ins = rng.integers(0, n_obj, n_in).astype(np.int32), rng.integers(0, n_obj, n_in).astype(np.int32)
    of, os_ = rng.integers(0, n_obj, n_out).astype(np.int32), rng.integers(0, n_obj, n_out).astype(np.int32)
    of[:2], os_[:2] = n_obj - 1, 0  # the last object (ragged quad / chunk / panel) on both sides
    a = synth.random_vector(n_obj, n_in)
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    u = ctx.matvec(d(D), None, d(of), d(os_), d(inf), d(ins), d(a), G.gvt_kernel_terms(G.RANKING)).cpu().numpy()
    st = ctx.stats()
    assert st["kinds"]["gemv"]["count"] > 0
    ref = O.gvt_matvec(O.kernel_terms(G.RANKING), D, None, of, os_, inf, ins, a)
    assert rel(u, ref) <= 1e-5, rel(u, ref)
