"""Bitwise check of improved.cdft_rows against the oracle at one size.  usage: parity_quick.py log2n batch [f64]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import parity  # noqa: E402
from paper_1301_0763_b200 import improved  # noqa: E402

lg, B = int(sys.argv[1]), int(sys.argv[2])
rt = torch.float64 if len(sys.argv) > 3 and sys.argv[3] == "f64" else torch.float32
x = torch.view_as_complex(torch.randn((B, 1 << lg, 2), dtype=rt, device="cuda"))
y = improved.cdft_rows(x)
torch.cuda.synchronize()
print(lg, rt, parity.check_rows(x, y))
