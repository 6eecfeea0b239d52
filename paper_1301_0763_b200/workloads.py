"""Seeded synthetic inputs of the BASELINE.json configurations (no dataset is
named by the reference or BASELINE.json; these stand in with the stated shapes,
sizes and value distributions -- SURVEY.md §8(d)).

Every generator returns batch-major data (batch, N) -- the GPU-native layout;
``.T`` gives the reference's (N, batch) layout.
"""

import numpy as np

CONFIGS = {
    1: dict(N=1 << 10, batch=64, dtype="complex128", desc="complex fp64, N=2^10, batch 64, re/im U[-1,1) seed 0"),
    2: dict(N=1 << 12, batch=16384, dtype="complex64", desc="complex fp32, N=2^12, batch 16384, re/im N(0,1)"),
    3: dict(N=1 << 16, batch=2048, dtype="complex64",
            desc="real fp32 (imag 0), N=2^16, batch 2048, 8 random sinusoids + 0.01 N(0,1)"),
    4: dict(N=1 << 20, batch=64, dtype="complex128", desc="complex fp64, N=2^20, batch 64, re/im U[-1,1)"),
    5: dict(N=1 << 14, batch=1 << 18, dtype="complex64",
            desc="complex fp32, N=2^14, batch 2^18 sharded over GPUs, re/im N(0,1) generated on device"),
}


def config1_input():
    """(N, batch) c128, re block then im block from default_rng(0) -- the same
    array is fed to the GPU and to the reference (tests/golden config1)."""
    rng = np.random.default_rng(0)
    N, B = 1 << 10, 64
    re = rng.uniform(-1.0, 1.0, (N, B))
    im = rng.uniform(-1.0, 1.0, (N, B))
    return re + 1j * im


def normal_rows(N, batch, seed, dtype=np.complex64):
    rng = np.random.default_rng(seed)
    re = rng.standard_normal((batch, N), dtype=np.float32 if dtype == np.complex64 else np.float64)
    im = rng.standard_normal((batch, N), dtype=re.dtype)
    out = np.empty((batch, N), dtype=dtype)
    out.real = re
    out.imag = im
    return out


def uniform_rows(N, batch, seed, dtype=np.complex128):
    rng = np.random.default_rng(seed)
    out = np.empty((batch, N), dtype=dtype)
    out.real = rng.uniform(-1.0, 1.0, (batch, N))
    out.imag = rng.uniform(-1.0, 1.0, (batch, N))
    return out


def sinusoid_params(N, batch, seed):
    """Per-signal frequencies f_i ~ U{1..N/2-1} and phases phi_i ~ U[0, 2pi), 8 each."""
    rng = np.random.default_rng(seed)
    f = rng.integers(1, N // 2, size=(batch, 8))
    phi = rng.uniform(0.0, 2.0 * np.pi, size=(batch, 8))
    return f, phi


def config3_rows_torch(N, batch, seed, device):
    """Config 3 input generated on the device: x(n) = sum_i sin(2 pi f_i n / N +
    phi_i) + 0.01 N(0,1), as complex64 with zero imaginary part.  The phase is
    reduced exactly (f_i n mod N in integers) before the fp64 sine."""
    import torch
    f, phi = sinusoid_params(N, batch, seed)
    n = torch.arange(N, device=device, dtype=torch.int64)
    fi = torch.as_tensor(f, device=device)
    ph = torch.as_tensor(phi, device=device)
    x = torch.zeros((batch, N), dtype=torch.float64, device=device)
    for i in range(8):
        k = (fi[:, i:i + 1] * n[None, :]) % N
        x += torch.sin(2.0 * np.pi * k.double() / N + ph[:, i:i + 1])
    g = torch.Generator(device=device).manual_seed(seed)
    x += 0.01 * torch.randn((batch, N), dtype=torch.float64, device=device, generator=g)
    return torch.complex(x.float(), torch.zeros_like(x, dtype=torch.float32))
