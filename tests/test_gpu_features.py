"""GPU checks of execution features that must not change results (-m gpu): CUDA-graph
replay of the CG loop, the CTA-pair vs single-CTA tensor-core GEMM, and the launch
accounting under graphs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O
import synth

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2009_01054_b200 as G


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def rel(x, ref):
    x, ref = np.asarray(x, np.float64), np.asarray(ref, np.float64)
    return np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-30)


@pytest.fixture(scope="module")
def ctx():
    c = G.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("cfg,kernel", [("C1", G.KRONECKER), ("C3", G.SYMMETRIC), ("C3", G.CARTESIAN),
                                        ("C2", G.KRONECKER)])
def test_graph_replay_is_bit_identical_to_eager(ctx, cfg, kernel):
    w = synth.config3(n=30_000, n_test=10) if cfg == "C3" else synth.by_name(cfg)
    D = ctx.gram(w.base, dev(w.Xd), gamma=w.gamma)
    T = None if w.Xt is None else ctx.gram(w.base, dev(w.Xt), gamma=w.gamma)
    terms = G.gvt_kernel_terms(kernel)
    f, s, y = dev(w.train_first), dev(w.train_second), dev(w.y)
    out = {}
    for graphs in (0, 1):
        ctx.set_option(G.OPT_GRAPHS, graphs)
        ctx.reset_stats()
        a, it, hist, code = ctx.fit(D, T, f, s, y, terms, w.lam, 12)
        st = ctx.stats()
        out[graphs] = (a.cpu().numpy(), it, hist, st["launches"])
    ctx.set_option(G.OPT_GRAPHS, 1)
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1] == 12
    assert np.array_equal(out[0][2], out[1][2])
    assert out[0][3] == out[1][3]  # replayed kernels are accounted per replay


def test_cta_pair_and_single_cta_gemm_agree_with_oracle(ctx):
    rng = np.random.default_rng(3)
    m, q = 700, 520          # ragged tile edges for both 128- and 256-row tiles
    D = O.gram(G.BASE_GAUSSIAN, rng.standard_normal((m, 12)), gamma=1 / 12).astype(np.float32)
    T = O.gram(G.BASE_GAUSSIAN, rng.standard_normal((q, 12)), gamma=1 / 12).astype(np.float32)
    inf, ins = rng.integers(0, m, 60000).astype(np.int32), rng.integers(0, q, 60000).astype(np.int32)
    of, os_ = rng.integers(0, m, 4000).astype(np.int32), rng.integers(0, q, 4000).astype(np.int32)
    a = synth.random_vector(11, 60000)
    kron = G.gvt_kernel_terms(G.KRONECKER)
    ref = O.gvt_matvec(O.kernel_terms(O.KRONECKER), D, T, of, os_, inf, ins, a)
    ctx.set_option(G.OPT_ENGINE, G.ENGINE_DENSE)
    try:
        for cta in (1, 2):
            for prec in (G.PREC_FP16X3, G.PREC_TF32X3):
                ctx.set_option(G.OPT_GEMM_CTA, cta)
                ctx.set_option(G.OPT_TC_PRECISION, prec)
                u = ctx.matvec(dev(D), dev(T), dev(of), dev(os_), dev(inf), dev(ins), dev(a), kron).cpu().numpy()
                assert rel(u, ref) <= 1e-5, (cta, prec, rel(u, ref))
    finally:
        ctx.set_option(G.OPT_GEMM_CTA, 2)
        ctx.set_option(G.OPT_TC_PRECISION, G.PREC_FP16X3)
        ctx.set_option(G.OPT_ENGINE, G.ENGINE_AUTO)


def test_bench_json_contract_on_c1():
    """bench.py prints one JSON line with the contract's keys (run on C1 to stay quick)."""
    import json
    import subprocess
    import sys
    root = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))
    out = subprocess.run([sys.executable, "bench.py", "--workload", "C1", "--steps", "2", "--warmup", "3",
                          "--no-cpu-baseline"], cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["e2e"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    g = d["gather_regime"]  # the sparse-engine gather leg (0.2 % density at C5 object counts)
    for leg in ("matvec", "predict"):
        assert g[leg]["engine"] == "sparse" and g[leg]["stage2_gather_ms"] > 0
        assert 0 < g[leg]["gather_frac_hbm"] < 2.0
    # SURVEY 8(d) breakdown fields: per-phase times and the standalone training matvec
    assert d["phases"]["fit_ms"] > 0 and d["phases"]["predict_ms"] > 0 and d["phases"]["gram_ms"] >= 0
    assert d["matvec"]["gpairs_per_s"] > 0 and d["matvec"]["runs"] == 5
    # per-config legs (C1-C4, every kernel) and the oracle's 1-core / explicit-K context legs
    runs = d["configs"]["runs"]
    assert [(r["config"], r["kernel"]) for r in runs] == [
        ("C1", "kronecker"), ("C2", "kronecker"), ("C3", "symmetric"), ("C3", "antisymmetric"), ("C3", "cartesian"),
        ("C4", "poly2d"), ("C4", "mlpk"), ("C4", "ranking")]
    assert all(r["ms_per_step"] > 0 and r["gpairs_per_s"] > 0 and r["us_per_iter_marginal"] > 0 for r in runs)
    assert all(r["frac_of_floor"] is not None for r in runs if r["config"] in ("C3", "C4"))
    o1 = d["configs"]["oracle_1core"]
    assert [r["config"] for r in o1] == ["C1", "C2", "C3"] and all(r["cores"] == 1 for r in o1)
    assert o1[0]["explicit_K"]["gpairs_per_s"] > 0
