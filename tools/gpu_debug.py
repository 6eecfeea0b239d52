import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
t0 = time.time()
def log(*a):
    print(f"[{time.time()-t0:7.2f}s]", *a, flush=True)
log("start")
import numpy as np
import torch
log("torch", torch.__version__, torch.cuda.is_available())
from paper_1301_0763_b200 import _native, improved
from oracle import oracle
log("imports ok")
for dt, lg in ((np.complex64, 4), (np.complex64, 8), (np.complex64, 12), (np.complex128, 10)):
    N = 1 << lg
    z = (np.random.default_rng(0).standard_normal((8, N)) + 1j).astype(dt)
    x = torch.from_numpy(z).cuda()
    y = improved.cdft_rows(x)
    torch.cuda.synchronize()
    ok = np.array_equal(y.cpu().numpy(), oracle.cdft_rows(z))
    log("N", N, dt.__name__, "bitwise" if ok else "MISMATCH")
