"""B200-native batched improved-QFT (arXiv 1301.0763).

Drop-in replacement for the reference package's transform entry points
(``quickfourier.improved`` / ``quickfourier.classical``) backed by hand-written
sm_100a CUDA kernels behind the C ABI in include/qft_b200.h.

    from paper_1301_0763_b200 import improved
    S = improved.cdft(z)            # same signature, dtype rule and errors

See DESIGN.md for the kernel design and INTEGRATION.md for the C ABI.
"""

from . import classical, counting, improved  # noqa: F401
from .counting import OpCounter, TrigTable, build_trig_table  # noqa: F401

__version__ = "0.1.0"
