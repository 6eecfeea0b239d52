"""Drop-in for ``quickfourier.classical`` (classical.py:134-167) -- the north
star's "classical QFT for comparison" entry point, on the GPU.

Same signatures, dtype rules, layouts and errors as the improved drop-in
(paper_1301_0763_b200.improved); the transforms run the classical recursion
(harmonic parity first, classical.py:64-129) in the warp-cooperative kernel of
csrc/qft_classical.cu, bit-identical to the reference.  ``counter`` receives
the exact classical op counts; ``table`` supplies the half-secants (the
classical footprint is the N/4 - 1 secant slots, counting.py:189-205).
"""

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
    return improved._exec_rows(x, out, table, counter, ALGO)


def rdft(values, table=None, counter=None):
    """Classical real-input DFT, k = 0..N/2 (classical.py:146-151)."""
    return improved._real(values, table, counter, "rdft", ALGO)


def dct0(values, table=None, counter=None):
    """Classical cosine transform; values are s(0)..s(N/2) (classical.py:134-138)."""
    return improved._real(values, table, counter, "dct0", ALGO)


def dst0(values, table=None, counter=None):
    """Classical sine transform; values are s(1)..s(N/2-1) (classical.py:140-144)."""
    return improved._real(values, table, counter, "dst0", ALGO)
