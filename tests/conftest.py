import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_fixtures.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests of the device path")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


def csr_from(g, name):
    from oracle import oracle as O
    rp = g[f"{name}.rp"]
    return O.Csr(len(rp) - 1, rp, g[f"{name}.cols"], g[f"{name}.vals"])


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.int64)
