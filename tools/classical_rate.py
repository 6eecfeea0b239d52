"""Throughput of the classical-QFT comparison path (classical.cdft_rows) next to
the improved one at the BASELINE config sizes, CUDA events on the current
stream.  usage: python tools/classical_rate.py [--json out.json]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1301_0763_b200 import classical, improved  # noqa: E402

CASES = [  # (log2N, dtype, batch)
    (10, torch.complex128, 64),
    (10, torch.complex64, 16384),
    (12, torch.complex64, 16384),
    (12, torch.complex128, 4096),
    (14, torch.complex64, 2048),
    (16, torch.complex64, 256),
    (20, torch.complex128, 8),
]


def rate(fn, x, reps):
    out = torch.empty_like(x)
    fn(x, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn(x, out=out)
    b.record()
    torch.cuda.synchronize()
    return x.shape[0] * reps / (a.elapsed_time(b) * 1e-3)


def main():
    rows = []
    g = torch.Generator(device="cuda").manual_seed(1)
    for lg, dt, B in CASES:
        N = 1 << lg
        rt = torch.float32 if dt == torch.complex64 else torch.float64
        x = torch.view_as_complex(torch.randn((B, N, 2), dtype=rt, device="cuda", generator=g))
        rc = rate(classical.cdft_rows, x, 2 if lg >= 16 else 5)
        ri = rate(improved.cdft_rows, x, 5)
        bpt = 2 * N * x.element_size()
        rows.append({"log2n": lg, "dtype": str(dt).split(".")[-1], "batch": B, "classical_tr_s": rc, "improved_tr_s": ri,
                     "classical_gbs": rc * bpt / 1e9, "improved_gbs": ri * bpt / 1e9})
        print(rows[-1], flush=True)
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
