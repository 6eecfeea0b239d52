"""Full-batch bitwise parity of device results against the CPU oracle --
TEST INFRASTRUCTURE ONLY (used by tests/ and by bench.py's post-timing parity
leg; never on the product path).

``check_rows(x, y)`` takes the device input rows x and the device result rows y
(batch-major (B, N) CUDA tensors), copies them to the host chunk by chunk and
compares every row of y with ``oracle.cdft_rows(x)`` byte for byte, on all host
threads.  Returns ``{"rows_checked", "mismatches", "first_mismatch", ...}``.
"""

import time

import numpy as np

from . import oracle


def check_rows(x, y, algo="improved", nthreads=None, chunk_bytes=512 << 20, row_range=None):
    import torch
    nthreads = nthreads or oracle.max_threads()
    B, N = x.shape
    r0, r1 = row_range or (0, B)
    per = max(1, chunk_bytes // (N * x.element_size()))
    bad, first, t0 = 0, None, time.perf_counter()
    hx = torch.empty((min(per, r1 - r0), N), dtype=x.dtype, pin_memory=True)
    hy = torch.empty_like(hx, pin_memory=True)
    for b0 in range(r0, r1, per):
        n = min(per, r1 - b0)
        hx[:n].copy_(x[b0:b0 + n])
        hy[:n].copy_(y[b0:b0 + n])
        want = oracle.cdft_rows(hx[:n].numpy(), algo=algo, nthreads=nthreads)
        got = hy[:n].numpy()
        eq = (got.view(np.uint8).reshape(n, -1) == want.view(np.uint8).reshape(n, -1)).all(axis=1)
        nb = int(n - eq.sum())
        if nb and first is None:
            first = b0 + int(np.argmin(eq))
        bad += nb
    return {"rows_checked": int(r1 - r0), "mismatches": int(bad), "first_mismatch": first,
            "oracle_threads": int(nthreads), "seconds": round(time.perf_counter() - t0, 2)}
