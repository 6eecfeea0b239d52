"""Drop-in for ``quickfourier.classical`` (classical.py:134-167) -- the north
star's "classical QFT for comparison" entry point, on the GPU.

Same signatures, dtype rules, layouts and errors as the improved drop-in
(paper_1301_0763_b200.improved); the transforms run the classical recursion
(harmonic parity first, classical.py:64-129) in the warp-cooperative kernel of
csrc/qft_classical.cu, bit-identical to the reference.  ``counter`` receives
the exact classical op counts; ``table`` supplies the half-secants (the
classical footprint is the N/4 - 1 secant slots, counting.py:189-205).
"""

import numpy as np

from . import _native, improved
from .counting import OpCounter  # noqa: F401  (reference-compatible import)

__all__ = ["cdft", "cdft_rows", "rdft", "dct0", "dst0"]

ALGO = _native.QFT_ALGO_CLASSICAL


def cdft(values, table=None, counter=None):
    """Classical complex DFT, reported for k = 0..N-1 (classical.py:156-167)."""
    if improved._is_torch(values):
        return improved._cdft_torch(values, table, counter, ALGO)
    return improved._cdft_numpy(values, table, counter, ALGO)


def cdft_rows(x, table=None, counter=None, out=None):
    """Batch-major (batch, N) CUDA tensor, transform along the last axis."""
    import torch
    if not (improved._is_torch(x) and x.is_cuda):
        raise TypeError("cdft_rows expects a CUDA torch.Tensor of shape (batch, N)")
    B, N = x.shape
    improved._check_n(N)
    dtype = np.float32 if x.dtype == torch.complex64 else np.float64
    if out is None:
        out = torch.empty((B, N), dtype=x.dtype, device=x.device)
    p = _native.plan(N.bit_length() - 1, 32 if dtype == np.float32 else 64, ALGO, x.device.index or 0)
    with p.lock:
        improved._apply_table(p, table, dtype, N, classical=True)
        p.exec_device(x.data_ptr(), out.data_ptr(), B, (x.stride(0), x.stride(1)), (out.stride(0), out.stride(1)),
                      torch.cuda.current_stream(x.device).cuda_stream)
    improved._count(counter, N, B, ALGO)
    return out


def rdft(values, table=None, counter=None):
    """Classical real-input DFT, k = 0..N/2 (classical.py:146-151)."""
    return improved._real(values, table, counter, "rdft", ALGO)


def dct0(values, table=None, counter=None):
    """Classical cosine transform; values are s(0)..s(N/2) (classical.py:134-138)."""
    return improved._real(values, table, counter, "dct0", ALGO)


def dst0(values, table=None, counter=None):
    """Classical sine transform; values are s(1)..s(N/2-1) (classical.py:140-144)."""
    return improved._real(values, table, counter, "dst0", ALGO)
