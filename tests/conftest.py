import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _ensure_built():
    """A fresh checkout has no libgvt.so (built artefacts are not committed): compile it (nvcc for
    sm_100a, no GPU needed) before the test modules import the binding, which fails loudly without it."""
    lib = os.path.join(ROOT, "paper_2009_01054_b200", "libgvt.so")
    if not os.path.exists(lib) and not os.environ.get("GVT_LIBRARY"):
        import importlib.util
        spec = importlib.util.spec_from_file_location("_gvt_build", os.path.join(ROOT, "paper_2009_01054_b200",
                                                                               "build.py"))
        b = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(b)
        b.build()


_ensure_built()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the sm_100a kernels through the C ABI)")
    config.addinivalue_line("markers", "slow: long-running (full-size workloads)")


def golden_path(name):
    return os.path.join(ROOT, "tests", "golden", name)


def load_golden_matrix(name):
    import numpy as np
    rows = []
    with open(golden_path(name)) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append([float(x) for x in line.split()])
    return np.array(rows)
