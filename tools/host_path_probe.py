"""Probe of the host-memory costs behind the numpy drop-in's e2e (run on the GPU box):
improved.cdft on a pageable (N, B) numpy array, cudaHostRegister/Unregister cost,
host memcpy bandwidth (1 and several threads), pinned H2D/D2H."""
import concurrent.futures as cf
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1301_0763_b200 import improved  # noqa: E402

res = {}
N, B = 4096, 16384
z = (np.random.default_rng(0).standard_normal((N, B), dtype=np.float32)).astype(np.complex64)
improved.cdft(z[:, :64])
for rep in range(3):
    t = time.perf_counter()
    y = improved.cdft(z)
    res[f"dropin_numpy_NB_s_{rep}"] = time.perf_counter() - t
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
try:
    cudart = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
except OSError:
    pass
if cudart is not None:
    buf = np.empty(N * B * 8, dtype=np.uint8)
    buf[::4096] = 1
    for rep in range(2):
        t = time.perf_counter()
        rc = cudart.cudaHostRegister(ctypes.c_void_p(buf.ctypes.data), ctypes.c_size_t(buf.nbytes), 0)
        t1 = time.perf_counter()
        rc2 = cudart.cudaHostUnregister(ctypes.c_void_p(buf.ctypes.data))
        res[f"host_register_512MB_s_{rep}"] = (t1 - t, time.perf_counter() - t1, rc, rc2)
src = np.ones(N * B * 8, dtype=np.uint8)
dst = np.empty_like(src)
for th in (1, 4, 8, 16):
    n = len(src)
    parts = [(i * n // th, (i + 1) * n // th) for i in range(th)]
    def cp(a):
        np.copyto(dst[a[0]:a[1]], src[a[0]:a[1]])
    with cf.ThreadPoolExecutor(th) as ex:
        list(ex.map(cp, parts))
        t = time.perf_counter()
        list(ex.map(cp, parts))
        res[f"memcpy_GBps_{th}thr"] = n / (time.perf_counter() - t) / 1e9
hp = torch.empty(N * B * 8, dtype=torch.uint8, pin_memory=True)
d = torch.empty(N * B * 8, dtype=torch.uint8, device="cuda")
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(hp, non_blocking=True); torch.cuda.synchronize()
    res["h2d_pinned_GBps"] = hp.numel() / (time.perf_counter() - t) / 1e9
    t = time.perf_counter(); hp.copy_(d, non_blocking=True); torch.cuda.synchronize()
    res["d2h_pinned_GBps"] = hp.numel() / (time.perf_counter() - t) / 1e9
hpg = torch.from_numpy(src)
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(hpg); torch.cuda.synchronize()
    res["h2d_pageable_GBps"] = hpg.numel() / (time.perf_counter() - t) / 1e9
print(json.dumps(res, indent=1))
