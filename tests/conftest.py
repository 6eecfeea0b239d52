import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


@pytest.fixture(scope="session")
def golden():
    arrays = np.load(os.path.join(GOLDEN, "golden.npz"))
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        meta = json.load(fh)
    return arrays, meta


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle
    oracle.lib()
    return oracle


def golden_input(N, B, dt, seed):
    """Same generator as tests/golden/make_golden.py:golden_input."""
    rng = np.random.default_rng(seed)
    re = rng.standard_normal((N, B))
    im = rng.standard_normal((N, B))
    return (re + 1j * im).astype(dt)


def config1_input():
    rng = np.random.default_rng(0)
    N, B = 1 << 10, 64
    re = rng.uniform(-1.0, 1.0, (N, B))
    im = rng.uniform(-1.0, 1.0, (N, B))
    return re + 1j * im


def sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bit_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()
