"""Operation counter and trigonometric-constant table of the drop-in API.

Mirrors the public surface of the reference's ``quickfourier.counting``
(/root/reference/pkg/src/quickfourier/counting.py:21-205) so that code written
against the reference keeps working after an import switch:

* ``OpCounter`` -- adds/muls tally.  The GPU path performs the reference's
  exact operation DAG, so it adds the closed-form counts
  (costmodel.py:69-71) times the batch size.
* ``TrigTable`` / ``build_trig_table`` -- constants keyed by reduced fraction,
  with the two-tier (wide then round once) and single-tier pipelines and the
  ``touched`` access log used by the footprint audits.

This module is host-side plan-building code; the device kernels read the
same constants from a level-ordered copy uploaded by the native plan.
"""

import math
from math import gcd

import numpy as np

# enough digits of pi that the 80-bit long-double tier is not limited by it
_PI_WIDE = np.longdouble("3.14159265358979323846264338327950288419716939937510")
PIPELINES = ("two_tier", "single_tier")


class OpCounter:
    """Tally of real additions and multiplications."""

    __slots__ = ("adds", "muls")

    def __init__(self):
        self.adds = 0
        self.muls = 0

    @property
    def flops(self):
        return self.adds + self.muls

    def reset(self):
        self.adds = 0
        self.muls = 0

    def __repr__(self):
        return f"OpCounter(adds={self.adds}, muls={self.muls})"


def _lg(N):
    return N.bit_length() - 1


def improved_cdft_counts(N):
    """(adds, muls) of one improved complex transform (costmodel.py:69-71)."""
    lg = _lg(N)
    return 3 * N * lg - 3 * N + 4, N * lg - 3 * N + 4


def improved_real_counts(kind, N):
    """(adds, muls) of improved.rdft / dct0 / dst0 (costmodel.py:72-82)."""
    lg = _lg(N)
    if kind == "rdft":
        return (3 * N * lg // 2 - 5 * N // 2 + 4, N * lg // 2 - 3 * N // 2 + 2)
    if kind == "dct0":
        return (3 * N * lg // 4 - 7 * N // 4 + lg + 3, N * lg // 4 - 3 * N // 4 + 1)
    return (3 * N * lg // 4 - 7 * N // 4 - lg + 3, N * lg // 4 - 3 * N // 4 + 1)


def classical_counts(kind, N):
    """(adds, muls) of classical.cdft/rdft/dct0/dst0, by replaying the integer
    structure of the classical recursion (classical.py:64-129; shared.py:21-72)."""
    from functools import lru_cache

    @lru_cache(None)
    def dct(n):
        if n == 2:
            return (2, 0)
        q = n // 4
        a, m = dct(n // 2)
        b, k = dct_odd(n)
        return (2 * q + a + b, m + k)

    @lru_cache(None)
    def dct_odd(n):
        if n == 4:
            return (0, 0)
        if n == 8:
            return (2, 1)
        q, q2 = n // 4, n // 8
        a, m = dct(n // 4)
        b, k = dct_odd(n // 2)
        return (2 * q2 + a + b + q, q + m + k)

    @lru_cache(None)
    def dst(n):
        if n == 4:
            return (0, 0)
        q = n // 4
        a, m = dst(n // 2)
        b, k = dst_odd(n)
        return (2 * (q - 1) + a + b, m + k)

    @lru_cache(None)
    def dst_odd(n):
        if n == 4:
            return (0, 0)
        q = n // 4
        a, m = dst(n // 2)
        return (a + (q - 2) + q, (q - 1) + m)

    def rdft(n):
        if n == 2:
            return (2, 0)
        a, m = dct(n)
        b, k = dst(n)
        return (2 * (n // 2 - 1) + a + b, m + k)

    if kind == "cdft":
        if N == 2:
            return (4, 0)
        a, m = rdft(N)
        return (2 * a + 2 * N - 4, 2 * m)
    if kind == "rdft":
        return rdft(N)
    if kind == "dct0":
        return dct(N)
    return dst(N)


def _cos_turns_wide(j, d, ftype):
    """cos(2 pi j/d) one tier above the working dtype."""
    if ftype is np.float32:
        return math.cos(2.0 * math.pi * (j / d))
    t = np.longdouble(j) / np.longdouble(d)
    return np.cos(2.0 * _PI_WIDE * t)


def _cos_turns_working(j, d, ftype):
    a = ftype(2.0) * ftype(np.pi) * (ftype(j) / ftype(d))
    return np.cos(a)


class TrigTable:
    """Half-secants 1/(2 cos(2 pi j/d)) keyed by reduced fraction j/d, plus
    the named eighth-turn cosine; logs which entries a run touched."""

    def __init__(self, dtype=np.float64, pipeline="two_tier"):
        if pipeline not in PIPELINES:
            raise ValueError(f"pipeline must be one of {PIPELINES}")
        self.dtype = np.dtype(dtype)
        if self.dtype.type not in (np.float32, np.float64):
            raise ValueError("working dtype must be float32 or float64")
        self.pipeline = pipeline
        self.half = self.dtype.type(0.5)
        self._cache = {}
        self.touched = set()

    def _compute(self, key):
        ft = self.dtype.type
        if key == ("cos8",):
            j, d = 1, 8
            c = _cos_turns_wide(j, d, ft) if self.pipeline == "two_tier" else _cos_turns_working(j, d, ft)
            return ft(c)
        _, j, d = key
        if self.pipeline == "two_tier":
            return ft(1.0 / (2.0 * _cos_turns_wide(j, d, ft)))
        return ft(1.0) / (ft(2.0) * _cos_turns_working(j, d, ft))

    def _lookup(self, key):
        v = self._cache.get(key)
        if v is None:
            v = self._compute(key)
            self._cache[key] = v
        self.touched.add(key)
        return v

    @staticmethod
    def key_for(n, N):
        g = gcd(n, N)
        j, d = n // g, N // g
        if d == 4:
            raise ValueError("half-secant undefined at a quarter turn")
        return ("sec", j, d)

    def half_secant(self, n, N):
        return self._lookup(self.key_for(n, N))

    def half_secants(self, N, ns):
        return np.array([self.half_secant(int(n), N) for n in ns], dtype=self.dtype)

    def eighth_cos(self):
        return self._lookup(("cos8",))

    def touched_count(self):
        return len(self.touched)

    def reset_log(self):
        self.touched = set()


def build_trig_table(algorithm, N, dtype=np.float64, pipeline="two_tier"):
    """Table pre-filled with the constants a full transform at N uses."""
    if algorithm not in ("classical", "improved"):
        raise ValueError("algorithm must be 'classical' or 'improved'")
    t = TrigTable(dtype=dtype, pipeline=pipeline)
    for m in range(1, N // 4):
        t.half_secant(m, N)
    if algorithm == "improved" and N >= 8:
        t.eighth_cos()
    t.reset_log()
    return t


def natural_constants(table, N):
    """The N/4 constants of a full improved transform at N from any table
    object with the TrigTable interface (reference or ours), in the native
    layout T[0]=cos8, T[m]=half_secant(m, N).  Reading them logs exactly the
    keys the reference's improved transform touches (test_improved.py:127-145)."""
    vals = [table.eighth_cos()] + [table.half_secant(m, N) for m in range(1, N // 4)]
    return np.asarray(vals, dtype=np.dtype(table.dtype))
