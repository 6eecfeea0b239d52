"""Variant check (tools only, on the GPU box): the library named by QFT_LIB
must give full-batch bitwise parity with the oracle at batch sizes that hit
every edge of the CTA / group scheduling, and repeated full-size runs must be
bitwise identical.  usage: QFT_LIB=variants/x.so python tools/vcheck.py [N] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle.parity import check_rows  # noqa: E402
from paper_1301_0763_b200 import improved  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
dt = torch.complex64 if len(sys.argv) <= 3 else getattr(torch, sys.argv[3])
g = torch.Generator(device="cuda").manual_seed(5)
ok = True
for B in (1, 2, 3, 4, 5, 7, 148, 443, 444, 445, 889, 1333, 2665, 16384):
    x = torch.randn((B, N), dtype=dt, device="cuda", generator=g)
    y = improved.cdft_rows(x)
    r = check_rows(x, y)
    if B == 16384:
        for i in range(reps):
            if not torch.equal(improved.cdft_rows(x).view(torch.float32), y.view(torch.float32)):
                r["repeat_mismatch"] = i
                ok = False
                break
    ok = ok and r["mismatches"] == 0
    print(f"N={N} B={B}: {r}", flush=True)
print("VCHECK", "OK" if ok else "FAIL", os.environ.get("QFT_LIB"))
