"""improved.cdft_rows throughput and HBM-roofline fraction across N (1 GiB of input per
launch, > L2), CUDA events.  usage: python tools/size_sweep.py [--json out.json] [--algo classical]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1301_0763_b200 import classical, improved  # noqa: E402


def main():
    algo = classical if "--algo" in sys.argv and sys.argv[sys.argv.index("--algo") + 1] == "classical" else improved
    try:
        peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6650.0
    rows = []
    for dt in (torch.complex64, torch.complex128):
        lo, hi = (int(sys.argv[sys.argv.index("--lg") + 1]), int(sys.argv[sys.argv.index("--lg") + 2])) if "--lg" in sys.argv else (5, 20)
        for lg in range(lo, hi + 1):
            N = 1 << lg
            es = 8 if dt == torch.complex64 else 16
            B = max(1, (1 << 30) // (N * es))
            rt = torch.float32 if dt == torch.complex64 else torch.float64
            x = torch.view_as_complex(torch.randn((B, N, 2), dtype=rt, device="cuda"))
            out = torch.empty_like(x)
            for _ in range(2):
                algo.cdft_rows(x, out=out)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 5
            a.record()
            for _ in range(reps):
                algo.cdft_rows(x, out=out)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
            gbs = 2 * B * N * es / (ms * 1e-3) / 1e9
            rows.append({"log2n": lg, "dtype": str(dt).split(".")[-1], "batch": B, "ms": ms, "tr_s": B / (ms * 1e-3),
                         "gbs": gbs, "frac": gbs / peak})
            print(f"{rows[-1]['dtype']:11s} 2^{lg:<2d} batch {B:8d}  {ms:8.3f} ms  {rows[-1]['tr_s']:14.0f} tr/s  "
                  f"{gbs:7.0f} GB/s  {100 * gbs / peak:5.1f} %", flush=True)
            del x, out
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
            json.dump({"peak_gbs": peak, "rows": rows}, fh, indent=1)


if __name__ == "__main__":
    main()
