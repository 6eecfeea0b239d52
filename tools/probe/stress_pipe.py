"""Stress check of the pipelined kernel (tools only): repeated full-size runs
must be bitwise identical (a shared-memory race or a missed mbarrier phase
shows up as run-to-run differences), and sampled rows must equal the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import sys
import numpy as np
import torch
from paper_1301_0763_b200 import improved
from oracle import oracle

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
g = torch.Generator(device="cuda").manual_seed(3)
for B in (16384, 4441, 889):
    x = torch.randn((B, 4096), dtype=torch.complex64, device="cuda", generator=g)
    ref = improved.cdft_rows(x)
    for r in range(reps):
        y = improved.cdft_rows(x)
        assert torch.equal(y.view(torch.float32), ref.view(torch.float32)), (B, r)
    idx = np.random.default_rng(B).integers(0, B, 48)
    z = x[idx].cpu().numpy()
    assert np.array_equal(ref[idx].cpu().numpy().view(np.uint8), oracle.cdft_rows(z).view(np.uint8)), B
    print(f"B={B}: {reps} runs bitwise identical, 48 sampled rows == oracle", flush=True)
