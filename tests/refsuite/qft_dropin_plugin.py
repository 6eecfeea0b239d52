"""pytest plugin: run the REFERENCE's own test modules against the drop-in.

Loaded with ``-p qft_dropin_plugin`` by tests/test_gpu_reference_suite.py.  It
imports the unmodified reference package installed under baseline/_ref (the
base contract's one offline install), then rebinds ``quickfourier.improved``
and ``quickfourier.classical`` -- in sys.modules and inside every already
imported quickfourier module (accuracy, costmodel, ...) -- to
paper_1301_0763_b200.improved / .classical.  Everything else the reference
tests use (the brute-force oracle reference.py, counting.TrigTable, taxonomy,
tree) stays the reference's own code, so the tests judge the GPU path exactly
as they judge the reference.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(ROOT, "baseline", "_ref")
sys.path.insert(0, ROOT)
sys.path.insert(1, REF)

import quickfourier  # noqa: E402  (the reference package)
from quickfourier import classical as _ref_classical  # noqa: E402
from quickfourier import improved as _ref_improved  # noqa: E402

from paper_1301_0763_b200 import _native  # noqa: E402
from paper_1301_0763_b200 import classical as _our_classical  # noqa: E402
from paper_1301_0763_b200 import improved as _our_improved  # noqa: E402

_native.load()  # fail loudly if the CUDA library is missing
_SWAP = {id(_ref_improved): _our_improved, id(_ref_classical): _our_classical}
sys.modules["quickfourier.improved"] = _our_improved
sys.modules["quickfourier.classical"] = _our_classical
for _name, _mod in list(sys.modules.items()):
    if _name == "quickfourier" or _name.startswith("quickfourier."):
        for _attr in ("improved", "classical"):
            _cur = getattr(_mod, _attr, None)
            if _cur is not None and id(_cur) in _SWAP:
                setattr(_mod, _attr, _SWAP[id(_cur)])


def pytest_report_header(config):
    return [f"quickfourier.improved -> {_our_improved.__file__}",
            f"quickfourier.classical -> {_our_classical.__file__}",
            f"reference package: {os.path.dirname(quickfourier.__file__)}"]
