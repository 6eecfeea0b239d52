"""Randomised parity stress (GPU): random sizes, precisions, batches, algorithms and entry
points for a time budget, every output row compared bit for bit with the oracle, and each
case run twice (run-to-run differences would expose a shared-memory race).
usage: python tools/stress_all.py [seconds] [seed]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402
from paper_1301_0763_b200 import classical, improved  # noqa: E402


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    t0, cases, rows = time.time(), 0, 0
    while time.time() - t0 < budget:
        lg = int(rng.integers(1, 18))
        f64 = bool(rng.integers(0, 2))
        algo = "classical" if rng.random() < 0.3 else "improved"
        mod = classical if algo == "classical" else improved
        kind = str(rng.choice(["cdft", "cdft", "cdft", "rdft", "dct0", "dst0"]))
        if kind == "dst0" and lg < 2:
            continue
        N = 1 << lg
        cap = max(1, min(3000, (1 << 24) // N))
        B = int(rng.integers(1, cap + 1))
        if kind == "cdft":
            dt = np.complex128 if f64 else np.complex64
            z = (rng.standard_normal((B, N)) + 1j * rng.standard_normal((B, N))).astype(dt)
            x = torch.from_numpy(z).cuda()
            y1 = mod.cdft_rows(x).cpu().numpy()
            y2 = mod.cdft_rows(x).cpu().numpy()
            want = oracle.cdft_rows(z, algo=algo, nthreads=oracle.max_threads())
        else:
            dt = np.float64 if f64 else np.float32
            n_vals = {"rdft": N, "dct0": N // 2 + 1, "dst0": N // 2 - 1}[kind]
            v = rng.standard_normal((n_vals, B)).astype(dt)
            y1 = getattr(mod, kind)(v)
            y2 = getattr(mod, kind)(v)
            want = getattr(oracle, kind)(v, algo=algo, nthreads=oracle.max_threads())
        same = y1.tobytes() == y2.tobytes()
        ok = y1.shape == want.shape and y1.tobytes() == np.ascontiguousarray(want).tobytes()
        if not (same and ok):
            print(f"MISMATCH algo={algo} kind={kind} N=2^{lg} f64={f64} B={B} repeat_equal={same} oracle_equal={ok}")
            sys.exit(1)
        cases += 1
        rows += B
    print(f"stress: {cases} cases, {rows} rows, all bit-identical to the oracle and to their repeat ({time.time() - t0:.0f}s)")


if __name__ == "__main__":
    main()
