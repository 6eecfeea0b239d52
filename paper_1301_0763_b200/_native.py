"""ctypes binding of libqftb200.so (the C ABI in include/qft_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_1301_0763_b200.build``).  There is no CPU fallback: if the
library or a CUDA device is missing, every transform raises ``RuntimeError``.
"""

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QFT_LIB") or os.path.join(_HERE, "libqftb200.so")  # QFT_LIB: A/B variants

QFT_PREC_F32 = 32
QFT_PREC_F64 = 64
QFT_ALGO_IMPROVED = 0
QFT_ALGO_CLASSICAL = 1
QFT_KIND_RDFT, QFT_KIND_DCT0, QFT_KIND_DST0 = 1, 2, 3

QFT_EINVAL = -1
QFT_EUNSUPPORTED = -2
QFT_ECUDA = -3


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("log2n", ctypes.c_int32),
        ("prec", ctypes.c_int32),
        ("algo", ctypes.c_int32),
        ("passes", ctypes.c_int32),
        ("kernel_launches", ctypes.c_int32),
        ("smem_bytes", ctypes.c_int32),
        ("threads_per_cta", ctypes.c_int32),
        ("ctas_per_sm", ctypes.c_int32),
        ("signals_per_cta", ctypes.c_int32),
        ("scratch_bytes", ctypes.c_int64),
    ]


# Every symbol include/qft_b200.h declares, with its ctypes signature.
_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
SIGNATURES = {
    "qft_version": (_I, []),
    "qft_plan_create": (_I, [ctypes.POINTER(_P), _I, _I, _I, _I]),
    "qft_plan_destroy": (_I, [_P]),
    "qft_plan_get_info": (_I, [_P, ctypes.POINTER(PlanInfo)]),
    "qft_plan_table": (_I, [_P, _P]),
    "qft_plan_set_table": (_I, [_P, _P]),
    "qft_exec_cdft": (_I, [_P, _P, _P, _I64, _I64, _I64, _I64, _I64, _P]),
    "qft_exec_cdft_host": (_I, [_P, _P, _P, _I64, _I64, _I64, _I64, _I64]),
    "qft_exec_real": (_I, [_P, _I, _P, _P, _I64, _P]),
    "qft_fill_normal": (_I, [_P, _P, _I64, _I64, ctypes.c_uint64, _P]),
    "qft_last_error": (ctypes.c_char_p, []),
}

_lib = None
_lock = threading.RLock()


def load():
    """Load libqftb200.so (raises RuntimeError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build the CUDA extension first "
                    "(python -c 'import __graft_entry__ as g; g.build()')")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error():
    return load().qft_last_error().decode(errors="replace")


def check(rc, what):
    if rc == 0:
        return
    msg = last_error()
    if rc == QFT_EINVAL:
        raise ValueError(f"{what}: {msg}")
    if rc == QFT_EUNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed ({rc}): {msg}")


class Plan:
    """Owning wrapper of a qft_plan* (immutable per (N, precision, algorithm, device))."""

    def __init__(self, log2n, prec, algo=QFT_ALGO_IMPROVED, device=0):
        self._lib = load()
        h = ctypes.c_void_p()
        check(self._lib.qft_plan_create(ctypes.byref(h), log2n, prec, algo, device), "qft_plan_create")
        self.handle = h
        self.log2n, self.N, self.prec, self.algo, self.device = log2n, 1 << log2n, prec, algo, device
        self.lock = threading.Lock()

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.qft_plan_destroy(h)
            except Exception:
                pass
            self.handle = None

    def info(self):
        info = PlanInfo()
        check(self._lib.qft_plan_get_info(self.handle, ctypes.byref(info)), "qft_plan_get_info")
        return info

    def table(self):
        import numpy as np
        dt = np.float32 if self.prec == QFT_PREC_F32 else np.float64
        out = np.zeros(max(self.N // 4, 1), dtype=dt)
        check(self._lib.qft_plan_table(self.handle, out.ctypes.data), "qft_plan_table")
        return out[: self.N // 4]

    def set_table(self, values):
        import numpy as np
        dt = np.float32 if self.prec == QFT_PREC_F32 else np.float64
        v = np.ascontiguousarray(values, dtype=dt)
        if v.shape != (self.N // 4,):
            raise ValueError("table must hold N/4 constants")
        check(self._lib.qft_plan_set_table(self.handle, v.ctypes.data), "qft_plan_set_table")

    def exec_device(self, d_in, d_out, batch, in_strides, out_strides, stream=0):
        check(self._lib.qft_exec_cdft(self.handle, d_in, d_out, batch, in_strides[0], in_strides[1],
                                      out_strides[0], out_strides[1], stream), "qft_exec_cdft")

    def exec_real(self, kind, d_in, d_out, nrows, stream=0):
        check(self._lib.qft_exec_real(self.handle, kind, d_in, d_out, nrows, stream), "qft_exec_real")

    def exec_host(self, h_in, h_out, batch, in_strides, out_strides):
        check(self._lib.qft_exec_cdft_host(self.handle, h_in, h_out, batch, in_strides[0], in_strides[1],
                                           out_strides[0], out_strides[1]), "qft_exec_cdft_host")

    def fill_normal(self, d_out, batch, first_index, seed, stream=0):
        check(self._lib.qft_fill_normal(self.handle, d_out, batch, first_index, seed, stream), "qft_fill_normal")


_plans = {}


def plan(log2n, prec, algo=QFT_ALGO_IMPROVED, device=0):
    """Plan cache keyed on (N, precision, algorithm, device) (SURVEY §5 config/flags)."""
    key = (log2n, prec, algo, device)
    p = _plans.get(key)
    if p is None:
        with _lock:
            p = _plans.get(key)
            if p is None:
                p = Plan(log2n, prec, algo, device)
                _plans[key] = p
    return p
