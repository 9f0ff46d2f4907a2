import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def face_fixed_mask(nx, ny, nz, axis=0, side=0):
    """All three dofs fixed on one domain face (same helper as the reference tests)."""
    mask = np.zeros((nz + 1, ny + 1, nx + 1, 3), dtype=bool)
    sl = [slice(None)] * 3
    sl[2 - axis] = 0 if side == 0 else -1
    mask[tuple(sl)] = True
    return mask.reshape(-1)


def rel_err(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = max(float(np.abs(b).max()), 1e-300)
    return float(np.abs(a - b).max()) / den
