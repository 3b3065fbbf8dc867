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


_ENTRY_LOG = os.environ.get("HX_ENTRY_LOG")


def close(a, b, tol, floor=1e-8, entry_tol=None, tag=""):
    """Parity check: the norm-wise relative error < tol AND every entry within
    entry_tol (default 100 tol) of the reference, relative to |b_i| + floor * max|b|
    (so small-magnitude entries such as far-field velocities cannot hide behind the
    norm).  HX_ENTRY_LOG=path appends the measured pair to a JSON-lines file."""
    r = rel(a, b)
    ee = entry_err(a, b, floor=floor)
    if _ENTRY_LOG:
        import json

        with open(_ENTRY_LOG, "a") as f:
            f.write(json.dumps({"tag": tag, "tol": tol, "rel": r, "entry": ee, "floor": floor}) + "\n")
    et = 100.0 * tol if entry_tol is None else entry_tol
    assert r < tol, f"{tag}: norm-wise relative error {r:.3e} >= {tol:.1e}"
    assert ee < et, f"{tag}: per-entry error {ee:.3e} >= {et:.1e} (floor {floor:.0e} max|b|)"
