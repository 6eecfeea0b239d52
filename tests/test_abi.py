"""C-ABI library: loads and exports every symbol include/qft_b200.h declares;
host-side argument validation mirrors the reference.  CPU only (no compute)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT


def header_symbols():
    src = open(os.path.join(ROOT, "include", "qft_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(qft_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1301_0763_b200 import _native
    lib = _native.load()
    syms = header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.SIGNATURES), "ctypes table out of sync with the header"
    assert lib.qft_version() == 100


def test_validation_before_device_work():
    from paper_1301_0763_b200 import improved
    with pytest.raises(ValueError, match="power of two"):
        improved.cdft(np.zeros(6, dtype=np.complex128))
    with pytest.raises(ValueError, match="power of two"):
        improved.cdft(np.zeros(1, dtype=np.complex64))


def test_plan_create_rejects_bad_arguments():
    import ctypes
    from paper_1301_0763_b200 import _native
    lib = _native.load()
    h = ctypes.c_void_p()
    assert lib.qft_plan_create(ctypes.byref(h), 0, 32, 0, 0) == _native.QFT_EINVAL
    assert lib.qft_plan_create(ctypes.byref(h), 10, 16, 0, 0) == _native.QFT_EINVAL
    assert "prec" in _native.last_error()


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1301_0763_b200 import improved
    with pytest.raises(RuntimeError):
        improved.cdft(np.ones(64, dtype=np.complex64))


def test_classical_validation_before_device_work():
    from paper_1301_0763_b200 import classical
    with pytest.raises(ValueError):
        classical.cdft(np.zeros(12))
