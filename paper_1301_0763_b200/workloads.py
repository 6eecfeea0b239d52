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


# input seed of each configuration (bench.py, the -m gpu config tests and the
# reference-generated fixtures of tests/golden/make_golden.py all use these)
SEEDS = {1: 0, 2: 2, 3: 3, 4: 4, 5: 5}


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


def uniform_rows(N, batch, seed, dtype=np.complex128, first=0):
    """Rows [first, first + batch) of re/im ~ U[-1, 1); every row is keyed on
    (seed, global row index), so any slice (a shard, a sampled row) regenerates
    on its own."""
    out = np.empty((batch, N), dtype=dtype)
    for r in range(batch):
        rng = np.random.default_rng([seed, first + r])
        out[r].real = rng.uniform(-1.0, 1.0, N)
        out[r].imag = rng.uniform(-1.0, 1.0, N)
    return out


def _sinusoid_rows(N, first, rows, seed, table):
    sin_t, cos_t = table
    n = np.arange(N, dtype=np.int64)
    x = np.empty((rows, N), dtype=np.float64)
    for r in range(rows):
        rng = np.random.default_rng([seed, first + r])
        f = rng.integers(1, N // 2, size=8)
        phi = rng.uniform(0.0, 2.0 * np.pi, size=8)
        acc = 0.01 * rng.standard_normal(N)
        for i in range(8):
            k = (f[i] * n) % N  # phase reduced exactly in integers
            # sin(2 pi k/N + phi) = sin(2 pi k/N) cos(phi) + cos(2 pi k/N) sin(phi)
            acc += sin_t[k] * np.cos(phi[i]) + cos_t[k] * np.sin(phi[i])
        x[r] = acc
    return x


def config3_rows(N, rows, first=0, seed=3, threads=None):
    """Config 3 input, rows [first, first + rows): x(n) = sum_{i<8} sin(2 pi f_i n/N
    + phi_i) + 0.01 N(0,1), f_i ~ U{1..N/2-1}, phi_i ~ U[0, 2pi), every row keyed
    on (seed, global row index) so any slice regenerates on its own; complex64
    with zero imaginary part (a real fp32 signal through cdft)."""
    import concurrent.futures as cf
    import os
    ang = 2.0 * np.pi * np.arange(N) / N
    table = (np.sin(ang), np.cos(ang))
    threads = threads or min(16, os.cpu_count() or 1)
    step = max(1, (rows + threads - 1) // threads)
    parts = [(r0, min(step, rows - r0)) for r0 in range(0, rows, step)]
    with cf.ThreadPoolExecutor(len(parts) or 1) as ex:
        outs = list(ex.map(lambda a: _sinusoid_rows(N, first + a[0], a[1], seed, table), parts))
    out = np.zeros((rows, N), dtype=np.complex64)
    if outs:
        out.real = np.concatenate(outs, 0)
    return out


def config3_rows_torch(N, batch, seed, device):
    """config3_rows uploaded to a CUDA device (generated on the host)."""
    import torch
    return torch.from_numpy(config3_rows(N, batch, 0, seed)).to(device)


# ---------------------------------------------------------------- keyed generator
# numpy twin of qft_fill_normal (paper_1301_0763_b200/csrc/qft_capi.cu): the same
# splitmix64 keys and the same sequence of IEEE double ops (numpy ufuncs round
# each op once, like the __d*_rn intrinsics), so every value is bit-identical to
# the device generator -- config-2 / config-5 rows can be regenerated on the host.
_GEN_LN = [float.fromhex(h) for h in (
    "0x1.0000000000000p+0", "0x1.5555555555555p-2", "0x1.999999999999ap-3", "0x1.2492492492492p-3",
    "0x1.c71c71c71c71cp-4", "0x1.745d1745d1746p-4", "0x1.3b13b13b13b14p-4", "0x1.1111111111111p-4",
    "0x1.e1e1e1e1e1e1ep-5", "0x1.af286bca1af28p-5", "0x1.8618618618618p-5", "0x1.642c8590b2164p-5")]
_GEN_SIN = [float.fromhex(h) for h in (
    "0x1.0000000000000p+0", "-0x1.5555555555555p-3", "0x1.1111111111111p-7", "-0x1.a01a01a01a01ap-13",
    "0x1.71de3a556c734p-19", "-0x1.ae64567f544e4p-26", "0x1.6124613a86d09p-33", "-0x1.ae7f3e733b81fp-41",
    "0x1.952c77030ad4ap-49", "-0x1.2f49b46814157p-57", "0x1.71b8ef6dcf572p-66", "-0x1.761b41316381ap-75")]
_GEN_COS = [float.fromhex(h) for h in (
    "0x1.0000000000000p+0", "-0x1.0000000000000p-1", "0x1.5555555555555p-5", "-0x1.6c16c16c16c17p-10",
    "0x1.a01a01a01a01ap-16", "-0x1.27e4fb7789f5cp-22", "0x1.1eed8eff8d898p-29", "-0x1.93974a8c07c9dp-37",
    "0x1.ae7f3e733b81fp-45", "-0x1.6827863b97d97p-53", "0x1.e542ba4020225p-62", "-0x1.0ce396db7f853p-70")]
_SQRT2 = float.fromhex("0x1.6a09e667f3bcdp+0")
_LN2 = float.fromhex("0x1.62e42fefa39efp-1")
_HALF_PI = float.fromhex("0x1.921fb54442d18p+0")


def _splitmix64(z):
    z = z + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _gen_ln(u):
    b = u.view(np.uint64)
    e = ((b >> np.uint64(52)) & np.uint64(0x7FF)).astype(np.int64) - 1023
    m = ((b & np.uint64(0x000FFFFFFFFFFFFF)) | np.uint64(0x3FF0000000000000)).view(np.float64)
    big = m > _SQRT2
    m = np.where(big, m * 0.5, m)
    e = e + big
    s = (m - 1.0) / (m + 1.0)
    s2 = s * s
    p = np.full_like(s, _GEN_LN[11])
    for k in range(10, -1, -1):
        p = p * s2 + _GEN_LN[k]
    return e.astype(np.float64) * _LN2 + (s * p) * 2.0


def _gen_sincos2pi(u):
    t = u * 4.0
    qd = np.floor(t)
    f = t - qd
    x = f * _HALF_PI
    x2 = x * x
    ps = np.full_like(x, _GEN_SIN[11])
    pc = np.full_like(x, _GEN_COS[11])
    for k in range(10, -1, -1):
        ps = ps * x2 + _GEN_SIN[k]
        pc = pc * x2 + _GEN_COS[k]
    s = ps * x
    c = pc
    q = qd.astype(np.int64)
    sn = np.where(q == 0, s, np.where(q == 1, c, np.where(q == 2, -s, -c)))
    cs = np.where(q == 0, c, np.where(q == 1, -s, np.where(q == 2, -c, s)))
    return sn, cs


def keyed_normal_rows(N, rows, first, seed, dtype=np.complex64):
    """Rows [first, first + rows) of qft_fill_normal(seed): (rows, N) batch-major,
    re/im ~ N(0,1), bit-identical to the device generator."""
    with np.errstate(over="ignore"):
        b = np.arange(first, first + rows, dtype=np.uint64)[:, None]
        n = np.arange(N, dtype=np.uint64)[None, :]
        key = _splitmix64(np.uint64(seed) ^ _splitmix64(b * np.uint64(0x100000001B3) + n))
        k2 = _splitmix64(key)
    u1 = ((key >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = (k2 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    r = np.sqrt(-2.0 * _gen_ln(u1))
    sn, cs = _gen_sincos2pi(u2)
    out = np.empty((rows, N), dtype=dtype)
    out.real = r * cs
    out.imag = r * sn
    return out


def config_rows_device(c, rows=None, first=0, device="cuda"):
    """Rows [first, first + rows) of configuration c's input as a batch-major
    CUDA tensor: configs 2 / 5 from the device generator (qft_fill_normal),
    configs 1 / 3 / 4 generated on the host and uploaded."""
    import torch
    cfg = CONFIGS[c]
    N, seed = cfg["N"], SEEDS[c]
    rows = cfg["batch"] if rows is None else rows
    dev = torch.device(device)
    if c in (2, 5):
        from . import _native
        x = torch.empty((rows, N), dtype=torch.complex64, device=dev)
        p = _native.plan(N.bit_length() - 1, 32, _native.QFT_ALGO_IMPROVED, dev.index or 0)
        with torch.cuda.device(dev):
            p.fill_normal(x.data_ptr(), rows, first, seed, torch.cuda.current_stream(dev).cuda_stream)
        return x
    if c == 1:
        host = np.ascontiguousarray(config1_input().T[first:first + rows])
    elif c == 3:
        host = config3_rows(N, rows, first, seed)
    else:
        host = uniform_rows(N, rows, seed, np.complex128, first)
    return torch.from_numpy(host).to(dev)
