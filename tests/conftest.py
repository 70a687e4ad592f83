"""Shared test plumbing.

Markers: ``gpu`` tests need a B200 (they call the CUDA path through the C-ABI);
everything else runs on CPU.  The oracle (oracle/) is the checker; golden
fixtures (tests/golden/*.npz) hold the reference's own outputs.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def nodes_from_i64(words):
    from oracle.oracle import NODE_DTYPE

    return np.ascontiguousarray(words, dtype=np.int64).view(NODE_DTYPE)


def weights_sha(weights) -> str:
    """sha256 over every entry's arrays, as tests/golden/make_golden.py::gen_pipeline."""
    import hashlib

    h = hashlib.sha256()
    for e in weights.entries:
        names = ("filters", "bias") if hasattr(e, "filters") else ("scale", "shift", "mean", "var")
        for a in names:
            h.update(np.ascontiguousarray(np.asarray(getattr(e, a))).tobytes())
    return h.hexdigest()


def normwise_err(a, ref):
    """max|a - ref| / max|ref| (BASELINE.json north_star tolerance form)."""
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    scale = max(float(np.abs(ref).max()) if ref.size else 0.0, 1e-30)
    return float(np.abs(a - ref).max()) / scale if ref.size else 0.0


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o

    o.lib()
    return o
