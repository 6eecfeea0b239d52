"""Drop-in for ``quickfourier.classical`` (classical.py:134-167).

The classical QFT is the "for comparison" entry point of the north star and
the next row of SURVEY.md §8(f).  Its sm_100a kernel is not built yet, so the
transforms validate their arguments exactly like the reference and then raise
``NotImplementedError``; there is no CPU fallback by design.
"""

import numpy as np

from .counting import OpCounter  # noqa: F401  (reference-compatible import)

__all__ = ["cdft", "rdft", "dct0", "dst0"]


def _not_built(name):
    raise NotImplementedError(
        f"classical.{name} has no sm_100a kernel yet (SURVEY.md §8(f) rank 1); "
        "there is no CPU fallback by design")


def cdft(values, table=None, counter=None):
    z = np.asarray(values)
    N = z.shape[0] if z.ndim else 0
    if N < 2 or N & (N - 1):
        raise ValueError(f"periodization must be a power of two >= 2, got {N}")
    _not_built("cdft")


def rdft(values, table=None, counter=None):
    _not_built("rdft")


def dct0(values, table=None, counter=None):
    _not_built("dct0")


def dst0(values, table=None, counter=None):
    _not_built("dst0")
