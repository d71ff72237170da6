import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


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
