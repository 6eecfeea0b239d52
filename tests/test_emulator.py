"""Host emulation of the device phase functions (tests/emu/, test-only) must be
bit-identical to the oracle: validates the kernel's layout/index logic on CPU."""

import ctypes
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, bit_equal

EMU_DIR = os.path.join(ROOT, "tests", "emu")
EMU_LIB = os.path.join(EMU_DIR, "libkernel_emu.so")


@pytest.fixture(scope="module")
def emu():
    src = os.path.join(EMU_DIR, "kernel_emu.cpp")
    hdrs = [os.path.join(ROOT, "paper_1301_0763_b200", "csrc", f) for f in
            ("qft_common.cuh", "qft_lee.cuh", "qft_smem.cuh", "qft_large.cuh", "qft_large_plan.h", "qft_leaf.cuh")]
    newest = max(os.path.getmtime(p) for p in [src] + hdrs)
    if not os.path.exists(EMU_LIB) or os.path.getmtime(EMU_LIB) < newest:
        cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
        subprocess.check_call([cxx, "-O1", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off",
                               "-o", EMU_LIB, src])
    lib = ctypes.CDLL(EMU_LIB)
    for name in ("emu_cdft_f64", "emu_cdft_f32", "emu_large_f64", "emu_large_f32"):
        getattr(lib, name).argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long,
                                       ctypes.c_void_p]
    return lib


@pytest.mark.parametrize("dt", [np.complex128, np.complex64])
@pytest.mark.parametrize("lg", list(range(1, 15)))
def test_emulated_kernel_bitwise(emu, oracle_mod, dt, lg):
    """Single-pass kernel phases (N <= 2^14: top levels + 1024-cell units above 4096)."""
    N = 1 << lg
    rt = np.float32 if dt == np.complex64 else np.float64
    rng = np.random.default_rng(100 + lg)
    B = 2
    z = (rng.standard_normal((B, N)) + 1j * rng.standard_normal((B, N))).astype(dt)
    y = np.empty_like(z)
    T = oracle_mod.table(N, rt) if N >= 8 else np.zeros(2, rt)
    fn = emu.emu_cdft_f32 if dt == np.complex64 else emu.emu_cdft_f64
    assert fn(lg, z.ctypes.data, y.ctypes.data, B, T.ctypes.data) == 0
    assert bit_equal(y, oracle_mod.cdft_rows(z))


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("lg", [6, 9, 12, 13, 14, 15, 16, 18])
@pytest.mark.parametrize("kind", ["rdft", "dct0", "dst0"])
def test_emulated_real_modes_bitwise(emu, oracle_mod, dt, lg, kind):
    """improved.rdft/dct0/dst0 through the same phase functions (two real rows per lane)."""
    N, m = 1 << lg, 1 << (lg - 1)
    rl = {"rdft": N, "dct0": m + 1, "dst0": m - 1}[kind]
    rng = np.random.default_rng(lg)
    x = rng.standard_normal((4, rl)).astype(dt)
    fn = emu.emu_real_f32 if dt == np.float32 else emu.emu_real_f64
    fn.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p]
    T = oracle_mod.table(N, dt)
    if kind == "rdft":
        y = np.empty((4, m + 1), dtype=np.complex64 if dt == np.float32 else np.complex128)
    else:
        y = np.empty((4, rl), dtype=dt)
    assert fn({"rdft": 1, "dct0": 2, "dst0": 3}[kind], lg, x.ctypes.data, y.ctypes.data, 4, T.ctypes.data) == 0
    want = getattr(oracle_mod, kind)(np.ascontiguousarray(x.T)).T
    assert bit_equal(y, np.ascontiguousarray(want))


@pytest.mark.parametrize("dt", [np.complex128, np.complex64])
@pytest.mark.parametrize("lg", [13, 14, 15, 16, 17, 20])
def test_emulated_multipass_bitwise(emu, oracle_mod, dt, lg):
    """The multi-pass schedule (qft_large_plan.h task lists + qft_large.cuh phases)."""
    N = 1 << lg
    rt = np.float32 if dt == np.complex64 else np.float64
    rng = np.random.default_rng(200 + lg)
    z = (rng.standard_normal((1, N)) + 1j * rng.standard_normal((1, N))).astype(dt)
    y = np.empty_like(z)
    T = oracle_mod.table(N, rt)
    fn = emu.emu_large_f32 if dt == np.complex64 else emu.emu_large_f64
    assert fn(lg, z.ctypes.data, y.ctypes.data, 1, T.ctypes.data) == 0
    assert bit_equal(y, oracle_mod.cdft_rows(z))


# ---------------------------------------------------------------------------
# classical QFT, level-synchronous schedule (csrc/qft_classical_lv.cuh)
CL_EMU_LIB = os.path.join(EMU_DIR, "libclassical_emu.so")


@pytest.fixture(scope="module")
def cl_emu():
    src = os.path.join(EMU_DIR, "classical_emu.cpp")
    hdrs = [os.path.join(ROOT, "paper_1301_0763_b200", "csrc", f) for f in ("qft_common.cuh", "qft_classical_lv.cuh")]
    newest = max(os.path.getmtime(p) for p in [src] + hdrs)
    if not os.path.exists(CL_EMU_LIB) or os.path.getmtime(CL_EMU_LIB) < newest:
        cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
        subprocess.check_call([cxx, "-O1", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off",
                               "-o", CL_EMU_LIB, src])
    lib = ctypes.CDLL(CL_EMU_LIB)
    for name in ("emu_classical_f32", "emu_classical_f64"):
        getattr(lib, name).argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_long, ctypes.c_long, ctypes.c_void_p]
    return lib


@pytest.mark.parametrize("dt", [np.complex128, np.complex64])
@pytest.mark.parametrize("lg", list(range(5, 17)))
def test_emulated_classical_bitwise(cl_emu, oracle_mod, dt, lg):
    """Whole tree (sublog 0) and the large-N schedule cut into sub-trees of 2^sublog
    (cosine sub-tree roots of both kinds, D and O): bit-identical to the oracle's
    restatement of classical.py:64-129."""
    N = 1 << lg
    rt = np.float32 if dt == np.complex64 else np.float64
    rng = np.random.default_rng(300 + lg)
    z = (rng.standard_normal((2, N)) + 1j * rng.standard_normal((2, N))).astype(dt)
    want = oracle_mod.cdft_rows(z, algo="classical")
    T = oracle_mod.table(N, rt)
    fn = cl_emu.emu_classical_f32 if dt == np.complex64 else cl_emu.emu_classical_f64
    for sub in [0] + [s for s in (5, 6, 9, 11, 12) if s < lg]:
        y = np.empty_like(z)
        assert fn(lg, 0, sub, z.ctypes.data, y.ctypes.data, 2, 0, T.ctypes.data) == 0
        assert bit_equal(y, want), (lg, sub)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("lg", [5, 6, 9, 12, 14])
@pytest.mark.parametrize("kind", ["rdft", "dct0", "dst0"])
def test_emulated_classical_real_modes_bitwise(cl_emu, oracle_mod, dt, lg, kind):
    """classical.rdft/dct0/dst0 through the same level functions (two real rows per
    lane, an odd row count leaves the last lane half unused)."""
    N, m = 1 << lg, 1 << (lg - 1)
    rl = {"rdft": N, "dct0": m + 1, "dst0": m - 1}[kind]
    mode = {"rdft": 1, "dct0": 2, "dst0": 3}[kind]
    rng = np.random.default_rng(lg)
    x = rng.standard_normal((3, rl)).astype(dt)
    want = np.ascontiguousarray(getattr(oracle_mod, kind)(x.T.copy(), algo="classical").T)
    T = oracle_mod.table(N, dt)
    fn = cl_emu.emu_classical_f32 if dt == np.float32 else cl_emu.emu_classical_f64
    for sub in [0] + [s for s in (5, 8) if s < lg]:
        if kind == "rdft":
            out = np.empty((3, m + 1), dtype=np.complex64 if dt == np.float32 else np.complex128)
        else:
            out = np.empty((3, rl), dtype=dt)
        assert fn(lg, mode, sub, x.ctypes.data, out.ctypes.data, 2, 3, T.ctypes.data) == 0
        assert bit_equal(out, want), (lg, kind, sub)
