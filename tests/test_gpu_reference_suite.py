"""The reference's OWN test battery run against the drop-in on the GPU.

SURVEY.md §8(f) row 3: ``/root/reference/pkg/tests/test_improved.py``,
``test_classical.py`` and the parity criteria of ``test_acceptance.py``
(criterion 4: brute-force spectra of all four transforms, N = 4..4096, 20
trials, rel RMS <= 1e-11; criterion 5: constant footprint N/4 and N/4-1;
criterion 7: the fp32 accuracy experiment, improved within 2 % of classical,
growing with N, degraded by single-tier constants) run unmodified, with
``quickfourier.improved`` / ``quickfourier.classical`` rebound to
paper_1301_0763_b200's modules (tests/refsuite/qft_dropin_plugin.py).

The test modules are the reference's; ``build()`` copies them (together with
the pip-installed reference package) into the git-ignored baseline/_ref when
/root/reference is present, and that directory travels to the GPU box.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REFTESTS = os.path.join(ROOT, "baseline", "_ref", "reftests")

SELECT = [
    ("test_improved.py", None),
    ("test_classical.py", None),
    ("test_acceptance.py", "criterion_4 or criterion_5 or criterion_7"),
]


@pytest.mark.parametrize("module,kexpr", SELECT, ids=[m for m, _ in SELECT])
def test_reference_module_against_dropin(module, kexpr, tmp_path):
    path = os.path.join(REFTESTS, module)
    if not os.path.exists(path):
        pytest.skip("baseline/_ref/reftests not present (build() copies it where /root/reference exists)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests", "refsuite"), ROOT,
                                         os.path.join(ROOT, "baseline", "_ref")])
    cmd = [sys.executable, "-m", "pytest", path, "-q", "-p", "qft_dropin_plugin", "-p", "no:cacheprovider",
           "--rootdir", str(tmp_path), "-s"]
    if kexpr:
        cmd += ["-k", kexpr]
    r = subprocess.run(cmd, cwd=str(tmp_path), env=env, capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-3000:]
    assert "passed" in r.stdout and "failed" not in r.stdout
