"""Parity of the sm_100a kernels with the oracle (bit-identical), through the
C ABI and the drop-in API.  Run on a B200 with -m gpu."""

import numpy as np
import pytest

from conftest import bit_equal, config1_input, golden_input, sha

pytestmark = pytest.mark.gpu

ALL_LG = list(range(1, 21))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def _rows(torch, z):
    from paper_1301_0763_b200 import improved
    return improved.cdft_rows(torch.from_numpy(np.ascontiguousarray(z)).cuda()).cpu().numpy()


@pytest.mark.parametrize("dt", [np.complex64, np.complex128])
@pytest.mark.parametrize("lg", ALL_LG)
def test_rows_bitwise_vs_oracle(torch_cuda, oracle_mod, dt, lg):
    N = 1 << lg
    B = 37 if lg <= 10 else (9 if lg <= 12 else (3 if lg <= 16 else 1))
    rng = np.random.default_rng(10 * lg + (dt == np.complex64))
    z = (rng.standard_normal((B, N)) + 1j * rng.standard_normal((B, N))).astype(dt)
    assert bit_equal(_rows(torch_cuda, z), oracle_mod.cdft_rows(z))


@pytest.mark.parametrize("tag,dt", [("c128", np.complex128), ("c64", np.complex64)])
def test_golden_raw(golden, torch_cuda, tag, dt):
    from paper_1301_0763_b200 import improved
    arrays, _ = golden
    for lg in range(1, 11):
        N = 1 << lg
        got = improved.cdft(arrays[f"in_{tag}_{N}"])
        assert bit_equal(got, arrays[f"improved_{tag}_{N}"]), N


@pytest.mark.parametrize("tag,dt", [("c128", np.complex128), ("c64", np.complex64)])
def test_golden_digests(golden, torch_cuda, tag, dt):
    from paper_1301_0763_b200 import improved
    _, meta = golden
    for lg in range(11, 17):
        N = 1 << lg
        e = meta["cdft_sha256"][f"improved_{tag}_{N}"]
        z = golden_input(N, e["batch"], dt, e["seed"])
        assert sha(improved.cdft(z)) == e["sha256"], N


def test_known_answer_vectors(golden, torch_cuda):
    from paper_1301_0763_b200 import improved
    arrays, _ = golden
    z8 = arrays["kat_cdft8_in"]
    got = improved.cdft(z8)
    assert bit_equal(got, arrays["kat_cdft8_improved"])
    np.testing.assert_allclose(got, arrays["kat_cdft8_frozen"], rtol=0, atol=1e-13)
    assert bit_equal(improved.cdft(z8.astype(np.complex64)), arrays["kat_cdft8_improved_c64"])
    assert bit_equal(improved.cdft(np.array([1, 1j, -1, -1j])), arrays["kat_rot4_improved"])
    imp = np.zeros(16, dtype=np.complex128)
    imp[0] = 1
    assert bit_equal(improved.cdft(imp), arrays["kat_impulse16_improved"])


def test_config1_full_batch(golden, torch_cuda):
    """BASELINE config 1: c128, N=2^10, batch 64, U[-1,1) seed 0 -- bit-identical."""
    from paper_1301_0763_b200 import improved
    _, meta = golden
    z = config1_input()
    assert sha(z) == meta["config1"]["input_sha256"]
    assert sha(improved.cdft(z)) == meta["config1"]["improved_sha256"]


def test_plan_table_bit_parity(golden, torch_cuda):
    from paper_1301_0763_b200 import _native
    arrays, meta = golden
    for prec, tag in ((64, "f64"), (32, "f32")):
        for lg in range(3, 13):
            T = _native.plan(lg, prec).table()
            assert T.tobytes() == arrays[f"table_{tag}_{1 << lg}"].tobytes()
            assert sha(T) == meta["table_sha256"][f"{tag}_{1 << lg}"]


@pytest.mark.parametrize("shape", [(64,), (64, 1), (64, 5), (128, 2, 3), (16, 4, 1, 2)])
def test_reference_layouts(torch_cuda, oracle_mod, shape):
    from paper_1301_0763_b200 import improved
    rng = np.random.default_rng(len(shape))
    z = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    got = improved.cdft(z)
    assert got.shape == z.shape and got.dtype == np.complex128
    assert bit_equal(got, oracle_mod.cdft(z))
    # non-contiguous input views
    zt = np.asfortranarray(z)
    assert bit_equal(improved.cdft(zt), oracle_mod.cdft(z))


def test_dtype_rules(torch_cuda, oracle_mod):
    from paper_1301_0763_b200 import improved
    x = np.random.default_rng(1).standard_normal(32).astype(np.float32)
    out = improved.cdft(x)  # real float32 -> complex128 path (improved.py:142-143)
    assert out.dtype == np.complex128
    assert bit_equal(out, oracle_mod.cdft(x.astype(np.complex128)))
    z = x.astype(np.complex64)
    assert improved.cdft(z).dtype == np.complex64
    assert improved.cdft(list(x)).dtype == np.complex128


def test_input_not_mutated(torch_cuda):
    from paper_1301_0763_b200 import improved
    z = golden_input(256, 4, np.complex64, 5)
    keep = z.copy()
    improved.cdft(z)
    assert bit_equal(z, keep)


def test_counter_and_table(torch_cuda, oracle_mod):
    from paper_1301_0763_b200 import improved
    from paper_1301_0763_b200.counting import OpCounter, TrigTable, build_trig_table
    z = golden_input(64, 7, np.complex128, 9)
    c = OpCounter()
    improved.cdft(z, counter=c)
    assert (c.adds, c.muls) == (6748, 1372)  # N=64 x 7
    t = build_trig_table("improved", 64, np.float64)
    improved.cdft(z, table=t, counter=OpCounter())
    assert t.touched_count() == 16
    with pytest.raises(ValueError, match="does not match"):
        improved.cdft(z, table=TrigTable(dtype=np.float32))
    # a single-tier table changes the constants the kernel uses
    st = TrigTable(dtype=np.float64, pipeline="single_tier")
    got = improved.cdft(golden_input(4096, 2, np.complex128, 3), table=st)
    from paper_1301_0763_b200.counting import natural_constants
    want = oracle_mod.cdft(golden_input(4096, 2, np.complex128, 3),
                           T=natural_constants(TrigTable(np.float64, "single_tier"), 4096))
    assert bit_equal(got, want)
    # and the default table is restored afterwards
    z2 = golden_input(4096, 2, np.complex128, 4)
    assert bit_equal(improved.cdft(z2), oracle_mod.cdft(z2))


def test_reference_table_objects_accepted(torch_cuda, oracle_mod):
    """A TrigTable from the reference package (duck-typed) drives the kernel."""
    import sys
    import os
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):  # the GPU box: the pip-installed copy (baseline/_ref, built here)
        ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "quickfourier")):
        pytest.skip("reference package not present on this host")
    sys.path.insert(0, ref)
    from quickfourier.counting import build_trig_table as ref_build
    from paper_1301_0763_b200 import improved
    t = ref_build("improved", 256, np.float64)
    z = golden_input(256, 3, np.complex128, 2)
    assert bit_equal(improved.cdft(z, table=t), oracle_mod.cdft(z))
    assert t.touched_count() == 64


def test_torch_device_path_reference_layout(torch_cuda, oracle_mod):
    from paper_1301_0763_b200 import improved
    torch = torch_cuda
    z = golden_input(512, 6, np.complex64, 11)
    t = torch.from_numpy(z).cuda()
    out = improved.cdft(t)
    assert out.is_cuda and out.shape == t.shape
    assert bit_equal(out.cpu().numpy(), oracle_mod.cdft(z))


def test_batched_equals_single_and_empty(torch_cuda, oracle_mod):
    from paper_1301_0763_b200 import improved
    torch = torch_cuda
    z = golden_input(4096, 1, np.complex64, 12)[:, 0]
    one = improved.cdft(z)
    zz = np.stack([z] * 300)
    many = improved.cdft_rows(torch.from_numpy(zz).cuda()).cpu().numpy()
    assert all(bit_equal(many[i], one) for i in (0, 150, 299))
    empty = improved.cdft_rows(torch.empty((0, 64), dtype=torch.complex64, device="cuda"))
    assert empty.shape == (0, 64)


def test_special_values(torch_cuda, oracle_mod):
    """zeros (signed-zero bookkeeping), huge, tiny/denormal inputs: still bit-identical."""
    for dt in (np.complex64, np.complex128):
        N = 1024
        cases = [np.zeros((2, N)), -np.zeros((2, N)), np.full((2, N), 1e30), np.full((2, N), 1e-39)]
        rng = np.random.default_rng(0)
        m = rng.standard_normal((2, N))
        m[:, ::3] = 0.0
        cases.append(m)
        for c in cases:
            z = (c + 1j * c[::-1]).astype(dt)
            assert bit_equal(_rows(torch_cuda, z), oracle_mod.cdft_rows(z))


def test_large_batch_properties(torch_cuda):
    """Config-2 sized batch: linearity and Parseval (size-independent checks)."""
    torch = torch_cuda
    from paper_1301_0763_b200 import improved
    N, B = 4096, 16384
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((B, N), dtype=torch.complex64, device="cuda", generator=g)
    y = improved.cdft_rows(x)
    # Parseval: sum |X|^2 = N sum |x|^2 per row
    ex = (x.abs() ** 2).double().sum(1) * N
    ey = (y.abs() ** 2).double().sum(1)
    assert torch.allclose(ey, ex, rtol=1e-4)
    # agreement with torch.fft (fp32 accuracy of the reference algorithm)
    ref = torch.fft.fft(x.to(torch.complex128), dim=1)
    rel = ((y.to(torch.complex128) - ref).abs().pow(2).sum(1).sqrt() / ref.abs().pow(2).sum(1).sqrt()).max()
    assert rel.item() < 1e-6 * 12


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("lg", list(range(1, 17)) + [18])
@pytest.mark.parametrize("kind", ["rdft", "dct0", "dst0"])
def test_real_entry_points_bitwise(torch_cuda, oracle_mod, dt, lg, kind):
    """improved.rdft / dct0 / dst0 (improved.py:117-136) on the GPU, bit-identical;
    above 2^14 (fp32) / 2^13 (fp64) through the multi-pass path."""
    from paper_1301_0763_b200 import improved
    N = 1 << lg
    if kind == "dst0" and N < 4:
        pytest.skip("the sine transform needs N >= 4")
    n_vals = {"rdft": N, "dct0": N // 2 + 1, "dst0": N // 2 - 1}[kind]
    rng = np.random.default_rng(lg * 7 + len(kind))
    x = rng.standard_normal((n_vals, 5)).astype(dt)  # odd batch: the last lane pairs with nothing
    got = getattr(improved, kind)(x)
    want = getattr(oracle_mod, kind)(x)
    assert got.dtype == want.dtype and got.shape == want.shape
    assert bit_equal(got, want)
    one = getattr(improved, kind)(x[:, 2])
    assert bit_equal(one, want[:, 2])


def test_real_entry_points_counts_and_errors(torch_cuda):
    from paper_1301_0763_b200 import improved
    from paper_1301_0763_b200.counting import OpCounter
    c = OpCounter()
    improved.rdft(np.random.default_rng(0).uniform(-0.5, 0.5, 16), counter=c)
    assert (c.adds, c.muls) == (60, 10)   # the worked 16-point example (test_improved.py:81-87)
    c = OpCounter()
    improved.dct0(np.random.default_rng(0).uniform(-0.5, 0.5, 9), counter=c)
    assert (c.adds, c.muls) == (27, 5)
    c = OpCounter()
    improved.dst0(np.random.default_rng(0).uniform(-0.5, 0.5, 7), counter=c)
    assert (c.adds, c.muls) == (19, 5)
    with pytest.raises(ValueError):
        improved.rdft(np.zeros(12))
    with pytest.raises(ValueError):
        improved.dct0(np.zeros(4))
    with pytest.raises(ValueError):
        improved.dst0(np.zeros(2))
    d = improved.dct0(np.array([1.0, 0, 0, 0, 0, 0, 0, 0, 1.0]))  # test_cli.py:10-16
    assert np.array_equal(d, [2, 0, 2, 0, 2, 0, 2, 0, 2])
    assert improved.rdft(np.zeros(8, dtype=np.int64)).dtype == np.complex128


@pytest.mark.parametrize("dt", [np.complex64, np.complex128])
@pytest.mark.parametrize("lg", [1, 2, 3, 4, 5, 6, 8, 10, 12, 14, 15, 16])  # 15, 16: one CTA team per signal
def test_classical_cdft_bitwise(torch_cuda, oracle_mod, dt, lg):
    """classical.cdft (classical.py:156-167) on the GPU, bit-identical to the oracle."""
    from paper_1301_0763_b200 import classical
    N = 1 << lg
    rng = np.random.default_rng(lg + 50)
    z = (rng.standard_normal((N, 3)) + 1j * rng.standard_normal((N, 3))).astype(dt)
    got = classical.cdft(z)
    assert got.dtype == dt
    assert bit_equal(got, oracle_mod.cdft(z, algo="classical"))


def test_classical_golden_digests_and_semantics(golden, torch_cuda, oracle_mod):
    from paper_1301_0763_b200 import classical
    from paper_1301_0763_b200.counting import OpCounter, build_trig_table
    _, meta = golden
    for tag, dt in (("c128", np.complex128), ("c64", np.complex64)):
        for lg in (5, 9, 12):
            e = meta["cdft_sha256"][f"classical_{tag}_{1 << lg}"]
            z = golden_input(1 << lg, e["batch"], dt, e["seed"])
            assert sha(classical.cdft(z)) == e["sha256"]
    z = config1_input()
    assert sha(classical.cdft(z)) == meta["config1"]["classical_sha256"]
    c = OpCounter()
    classical.cdft(golden_input(64, 2, np.complex128, 3), counter=c)
    assert [c.adds, c.muls] == [2 * v for v in meta["classical_counts"]["cdft_64"]]
    t = build_trig_table("classical", 256, np.float64)
    classical.cdft(golden_input(256, 1, np.complex128, 3)[:, 0], table=t)
    assert t.touched_count() == 256 // 4 - 1   # classical footprint (test_acceptance.py criterion 5)


@pytest.mark.parametrize("kind", ["rdft", "dct0", "dst0"])
@pytest.mark.parametrize("lg", [3, 7, 11, 15])
def test_classical_real_entry_points(torch_cuda, oracle_mod, kind, lg):
    from paper_1301_0763_b200 import classical
    N = 1 << lg
    n_vals = {"rdft": N, "dct0": N // 2 + 1, "dst0": N // 2 - 1}[kind]
    for dt in (np.float32, np.float64):
        x = np.random.default_rng(lg).standard_normal((n_vals, 3)).astype(dt)
        assert bit_equal(getattr(classical, kind)(x), getattr(oracle_mod, kind)(x, algo="classical"))


def test_classical_config4_accuracy_comparison(torch_cuda, oracle_mod):
    """config 4's comparison: improved vs classical on the GPU at N=2^20 fp64."""
    torch = torch_cuda
    from paper_1301_0763_b200 import classical, improved, workloads
    z = workloads.uniform_rows(1 << 20, 2, seed=4)
    x = torch.from_numpy(z).cuda()
    yi = improved.cdft_rows(x).cpu().numpy()
    yc = classical.cdft_rows(x).cpu().numpy()
    assert bit_equal(yc[:1], oracle_mod.cdft_rows(z[:1], algo="classical"))
    ref = np.fft.fft(z, axis=1)
    ei = np.linalg.norm(yi - ref) / np.linalg.norm(ref)
    ec = np.linalg.norm(yc - ref) / np.linalg.norm(ref)
    assert ei < 1e-12 and ec < 1e-12


@pytest.mark.parametrize("dt", [np.complex64, np.complex128])
@pytest.mark.parametrize("lg", [13, 14])
def test_single_pass_and_multipass_agree(torch_cuda, oracle_mod, dt, lg, monkeypatch):
    """N = 2^13 / 2^14 run single-pass (top levels + 1024-cell units) where the
    working area fits; QFT_MULTIPASS=1 forces the multi-pass schedule.  Both are
    bit-identical to the oracle."""
    import torch
    from paper_1301_0763_b200 import _native
    N = 1 << lg
    prec = 32 if dt == np.complex64 else 64
    rng = np.random.default_rng(lg + prec)
    z = (rng.standard_normal((5, N)) + 1j * rng.standard_normal((5, N))).astype(dt)
    want = oracle_mod.cdft_rows(z)
    outs = {}
    for mp in ("0", "1"):
        monkeypatch.setenv("QFT_MULTIPASS", mp)
        p = _native.Plan(lg, prec)           # uncached: the variable is read at plan creation
        info = p.info()
        single = not (prec == 64 and lg == 14) and mp == "0"
        assert (info.passes == 1) == single, (mp, info.passes)
        x = torch.from_numpy(z).cuda()
        y = torch.empty_like(x)
        p.exec_device(x.data_ptr(), y.data_ptr(), 5, (N, 1), (N, 1))
        torch.cuda.synchronize()
        outs[mp] = y.cpu().numpy()
        assert bit_equal(outs[mp], want), mp


@pytest.mark.parametrize("B", [1, 2, 3, 4, 5, 7, 443, 444, 445, 887, 889, 1333, 2665])
def test_pipelined_kernel_batch_edges(torch_cuda, oracle_mod, B):
    """fp32 N=4096 runs the pipelined kernel (qft_pipe.cuh: two slot sets, TT = 3
    signals per batch, in-place A0 of batch i+1 during phase D of batch i).
    Batches around multiples of 3 x 148 exercise the partial last batch, CTAs
    with one / two / three iterations (prologue-only TMA, no refill) and a grid
    smaller than the SM count -- bit-identical to the oracle on every row."""
    N = 4096
    rng = np.random.default_rng(B)
    z = (rng.standard_normal((B, N)) + 1j * rng.standard_normal((B, N))).astype(np.complex64)
    got = _rows(torch_cuda, z)
    rows = np.unique(np.r_[np.arange(min(B, 8)), np.arange(max(0, B - 8), B), rng.integers(0, B, 16)])
    assert bit_equal(got[rows], oracle_mod.cdft_rows(z[rows]))


@pytest.mark.parametrize("lg,dt", [(12, np.complex64), (14, np.complex64), (16, np.complex64), (10, np.complex64)])
def test_misaligned_input_view(torch_cuda, oracle_mod, lg, dt):
    """A batch-major complex64 view at an odd element offset (8-byte, not
    16-byte, aligned): the C ABI routes it through its aligned scratch copy
    (TMA bulk copies and 16-byte loads need 16-byte alignment)."""
    torch = torch_cuda
    from paper_1301_0763_b200 import improved
    N, B = 1 << lg, 5
    rng = np.random.default_rng(lg)
    z = (rng.standard_normal((B, N)) + 1j * rng.standard_normal((B, N))).astype(dt)
    flat = torch.zeros(B * N + 1, dtype=torch.complex64, device="cuda")
    flat[1:] = torch.from_numpy(z.reshape(-1)).cuda()
    x = flat[1:].view(B, N)
    assert x.data_ptr() % 16 == 8
    got = improved.cdft_rows(x).cpu().numpy()
    assert bit_equal(got, oracle_mod.cdft_rows(z))


@pytest.mark.parametrize("lg,dt", [(12, np.complex64), (10, np.complex128), (16, np.complex64)])
def test_cuda_graph_capture_replay(torch_cuda, oracle_mod, lg, dt):
    """A cdft call captured into a CUDA graph (the C ABI skips its cross-call event
    protocol on a capturing stream) replays bit-identically, on fresh inputs."""
    torch = torch_cuda
    from paper_1301_0763_b200 import improved
    N = 1 << lg
    rng = np.random.default_rng(lg)
    tdt = torch.complex64 if dt == np.complex64 else torch.complex128
    x = torch.empty((7, N), dtype=tdt, device="cuda")
    y = torch.empty_like(x)
    improved.cdft_rows(x.normal_(), out=y)  # plan + scratch outside the capture
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        improved.cdft_rows(x, out=y)
    for _ in range(2):
        z = (rng.standard_normal((7, N)) + 1j * rng.standard_normal((7, N))).astype(dt)
        x.copy_(torch.from_numpy(z))
        g.replay()
        torch.cuda.synchronize()
        assert bit_equal(y.cpu().numpy(), oracle_mod.cdft_rows(z))


@pytest.mark.parametrize("dt,lg,B", [(np.complex64, 12, 16384), (np.complex64, 10, 1000), (np.complex128, 12, 700),
                                     (np.complex64, 13, 300), (np.complex128, 13, 40), (np.complex64, 14, 150),
                                     (np.complex64, 5, 333), (np.complex128, 6, 149), (np.complex64, 17, 5)])
def test_classical_level_schedule_full_batches(torch_cuda, dt, lg, B):
    """The level-synchronous classical kernels (qft_classical_lv.cuh): every row of
    whole batches -- more signals than resident CTAs, a ragged last wave, the
    whole-tree kernel (fp32 <= 2^13, fp64 <= 2^12) and the global-level + sub-tree
    schedule above -- bit-identical to the oracle's classical.py restatement."""
    torch = torch_cuda
    from oracle import parity
    from paper_1301_0763_b200 import classical
    N = 1 << lg
    rt = torch.float32 if dt == np.complex64 else torch.float64
    g = torch.Generator(device="cuda").manual_seed(lg * 1000 + B)
    x = torch.view_as_complex(torch.randn((B, N, 2), dtype=rt, device="cuda", generator=g))
    y = classical.cdft_rows(x)
    torch.cuda.synchronize()
    rep = parity.check_rows(x, y, algo="classical")
    assert rep["rows_checked"] == B and rep["mismatches"] == 0, rep


def test_classical_large_schedule_chunked_scratch(torch_cuda, oracle_mod, monkeypatch):
    """A scratch budget smaller than the batch's W0/W1 (QFT_CL_ARENA_MB): the large-N
    schedule runs the batch in chunks, complex and real entry points alike."""
    from paper_1301_0763_b200 import classical
    monkeypatch.setenv("QFT_CL_ARENA_MB", "3")   # 2^15 fp32: ~0.5 MB per signal -> 5 signals per chunk
    N = 1 << 15
    rng = np.random.default_rng(77)
    z = (rng.standard_normal((N, 13)) + 1j * rng.standard_normal((N, 13))).astype(np.complex64)
    assert bit_equal(classical.cdft(z), oracle_mod.cdft(z, algo="classical"))
    for kind, n_vals in (("rdft", N), ("dct0", N // 2 + 1), ("dst0", N // 2 - 1)):
        x = rng.standard_normal((n_vals, 27)).astype(np.float32)
        assert bit_equal(getattr(classical, kind)(x), getattr(oracle_mod, kind)(x, algo="classical")), kind


def test_classical_recursive_kernel_still_matches(torch_cuda, oracle_mod):
    """N < 32 is served by the warp-recursive kernel (qft_classical.cu, first half)."""
    from paper_1301_0763_b200 import classical
    for lg in (1, 2, 3, 4):
        z = (np.random.default_rng(lg).standard_normal((1 << lg, 70)) + 0j).astype(np.complex128)
        assert bit_equal(classical.cdft(z), oracle_mod.cdft(z, algo="classical"))


@pytest.mark.parametrize("dt", [np.complex64, np.complex128])
@pytest.mark.parametrize("lg", [6, 7, 8, 9, 10, 11, 13])
def test_small_sizes_full_batches_bitwise(torch_cuda, dt, lg):
    """The phased-unit schedule of N <= 2048 (Lee-32 chunks of all signals of a CTA
    iteration flat over the threads, several resident CTAs) and the one-signal-per-
    iteration 2^13 / fp64 2^12 configurations: every row of batches that leave the last
    iteration ragged, that are smaller than the resident CTAs (signals per iteration
    lowered at launch), and that give every CTA several iterations."""
    torch = torch_cuda
    from oracle import parity
    from paper_1301_0763_b200 import improved
    N = 1 << lg
    rt = torch.float32 if dt == np.complex64 else torch.float64
    g = torch.Generator(device="cuda").manual_seed(lg)
    for B in (1, 2, 7, 147, 449, 1501, 20011 if lg <= 9 else 5003):
        x = torch.view_as_complex(torch.randn((B, N, 2), dtype=rt, device="cuda", generator=g))
        y = improved.cdft_rows(x)
        torch.cuda.synchronize()
        rep = parity.check_rows(x, y)
        assert rep["rows_checked"] == B and rep["mismatches"] == 0, (lg, B, rep)


@pytest.mark.parametrize("kind", ["rdft", "dct0", "dst0"])
@pytest.mark.parametrize("lg", [6, 8, 10, 11])
def test_small_sizes_real_modes_many_rows(torch_cuda, oracle_mod, kind, lg):
    """Real entry points through the phased units: odd row counts (the last vec2 lane
    half unused) over several CTA iterations."""
    from paper_1301_0763_b200 import improved
    N = 1 << lg
    n_vals = {"rdft": N, "dct0": N // 2 + 1, "dst0": N // 2 - 1}[kind]
    for dt in (np.float32, np.float64):
        x = np.random.default_rng(lg).standard_normal((n_vals, 1237)).astype(dt)
        assert bit_equal(getattr(improved, kind)(x), getattr(oracle_mod, kind)(x))
