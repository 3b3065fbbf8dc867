import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")


def golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def rel(a, b):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture
def gold():
    return golden


def entry_err(a, b, floor=1e-6):
    """Largest per-entry error relative to |b_i| + floor * max|b| (an entry-wise check with
    an absolute floor: a norm-wise error can hide large errors in small entries)."""
    a = np.asarray(a, float).reshape(-1)
    b = np.asarray(b, float).reshape(-1)
    if b.size == 0:
        return 0.0
    s = float(np.max(np.abs(b)))
    if s == 0.0:
        return float(np.max(np.abs(a)))
    return float(np.max(np.abs(a - b) / (np.abs(b) + floor * s)))
