"""Golden values of the reference's fp32 accuracy harness
(quickfourier.accuracy, /root/reference/pkg/src/quickfourier/accuracy.py:77-116),
produced by running the REFERENCE itself in the build container:
    python tests/golden/make_accuracy_golden.py
The GPU harness (paper_1301_0763_b200.accuracy) runs the same Philox inputs
through bit-identical transforms, so its mean errors agree with these up to
the rounding of the fp64 brute-force oracle (tests/test_accuracy_harness.py)."""

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from quickfourier import accuracy  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "accuracy_golden.json")


def main():
    rows = []
    for algo, N, trials, seed, pipe in [("improved", 256, 20, 3, "two_tier"), ("classical", 256, 20, 3, "two_tier"),
                                        ("improved", 1024, 10, 1234, "two_tier"),
                                        ("improved", 1024, 10, 1234, "single_tier"),
                                        ("classical", 2048, 8, 7, "two_tier")]:
        r = accuracy.run_accuracy(algo, N, trials=trials, seed=seed, pipeline=pipe)
        rows.append({"algorithm": algo, "N": N, "trials": trials, "seed": seed, "pipeline": pipe,
                     "mean_rel_rms_error": r.mean_rel_rms_error})
    sig = accuracy.random_signal(16, seed=7, trial=3)
    real = accuracy.random_real_batch(5, seed=9, trials=2)
    out = {"rows": rows,
           "random_signal_16_7_3": [[float(v.real), float(v.imag)] for v in sig],
           "random_real_batch_5_9_2": real.tolist()}
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
