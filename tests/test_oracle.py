"""The CPU parity oracle (oracle/) pinned against fixtures produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import bit_equal, config1_input, golden_input, sha


@pytest.mark.parametrize("tag,dt", [("f64", np.float64), ("f32", np.float32)])
def test_tables_bitwise(golden, oracle_mod, tag, dt):
    arrays, meta = golden
    for lg in range(3, 21):
        N = 1 << lg
        T = oracle_mod.table(N, dt)
        if lg <= 12:
            assert bit_equal(T, arrays[f"table_{tag}_{N}"]), N
        assert sha(T) == meta["table_sha256"][f"{tag}_{N}"], N


def test_single_tier_table(golden, oracle_mod):
    arrays, _ = golden
    assert bit_equal(oracle_mod.table(4096, np.float64, "single_tier"), arrays["table_f64_single_4096"])


def test_eighth_cos_equals_half_secant_eighth(oracle_mod):
    # the kernels may use either; the reference's two values are bit-equal
    for dt in (np.float64, np.float32):
        for N in (8, 64, 4096):
            T = oracle_mod.table(N, dt)
            assert T[0] == T[N // 8]


@pytest.mark.parametrize("tag,dt", [("c128", np.complex128), ("c64", np.complex64)])
def test_cdft_raw_golden_bitwise(golden, oracle_mod, tag, dt):
    arrays, _ = golden
    for lg in range(1, 11):
        N = 1 << lg
        z = arrays[f"in_{tag}_{N}"]
        assert bit_equal(oracle_mod.cdft(z), arrays[f"improved_{tag}_{N}"]), N


@pytest.mark.parametrize("tag,dt", [("c128", np.complex128), ("c64", np.complex64)])
def test_cdft_digest_golden(golden, oracle_mod, tag, dt):
    _, meta = golden
    for lg in range(11, 17):
        N = 1 << lg
        e = meta["cdft_sha256"][f"improved_{tag}_{N}"]
        z = golden_input(N, e["batch"], dt, e["seed"])
        assert sha(oracle_mod.cdft(z, nthreads=4)) == e["sha256"], N


@pytest.mark.parametrize("tag,dt", [("c128", np.complex128), ("c64", np.complex64)])
def test_classical_digest_golden(golden, oracle_mod, tag, dt):
    _, meta = golden
    for lg in range(1, 13):
        N = 1 << lg
        e = meta["cdft_sha256"][f"classical_{tag}_{N}"]
        z = golden_input(N, e["batch"], dt, e["seed"])
        assert sha(oracle_mod.cdft(z, algo="classical")) == e["sha256"], N


def test_known_answer_vectors(golden, oracle_mod):
    arrays, _ = golden
    z8 = arrays["kat_cdft8_in"]
    got = oracle_mod.cdft(z8)
    assert bit_equal(got, arrays["kat_cdft8_improved"])
    # the reference's frozen 50-digit values (test_reference.py:206-209), atol 1e-13
    np.testing.assert_allclose(got, arrays["kat_cdft8_frozen"], rtol=0, atol=1e-13)
    assert bit_equal(oracle_mod.cdft(z8.astype(np.complex64)), arrays["kat_cdft8_improved_c64"])
    rot = np.array([1, 1j, -1, -1j])
    got = oracle_mod.cdft(rot)
    assert bit_equal(got, arrays["kat_rot4_improved"])
    np.testing.assert_allclose(got, [0, 4, 0, 0], atol=1e-14)
    imp = np.zeros(16, dtype=np.complex128)
    imp[0] = 1
    got = oracle_mod.cdft(imp)
    assert bit_equal(got, arrays["kat_impulse16_improved"])
    assert np.all(got == 1)


def test_config1_digest(golden, oracle_mod):
    _, meta = golden
    z = config1_input()
    assert sha(z) == meta["config1"]["input_sha256"]
    assert sha(oracle_mod.cdft(z)) == meta["config1"]["improved_sha256"]
    assert sha(oracle_mod.cdft(z, algo="classical")) == meta["config1"]["classical_sha256"]


def test_batched_equals_single(oracle_mod):
    z = golden_input(256, 5, np.complex64, 3)
    full = oracle_mod.cdft(z)
    for b in range(5):
        assert bit_equal(oracle_mod.cdft(z[:, b]), full[:, b])


def test_oracle_validation():
    from oracle import oracle
    with pytest.raises(ValueError):
        oracle.cdft(np.zeros(6, dtype=np.complex128))
    with pytest.raises(ValueError):
        oracle.cdft(np.zeros(1, dtype=np.complex128))


# ---- fixtures added in round 2 (tests/golden/make_golden.py sections 6-8) ----

@pytest.mark.parametrize("tag,dt", [("c128", np.complex128), ("c64", np.complex64)])
def test_cdft_large_digest_golden(golden, oracle_mod, tag, dt):
    """improved cdft N = 2^17 .. 2^20 against the reference's own output."""
    _, meta = golden
    for lg in range(17, 21):
        N = 1 << lg
        e = meta["cdft_sha256"][f"improved_{tag}_{N}"]
        z = golden_input(N, e["batch"], dt, e["seed"])
        assert sha(oracle_mod.cdft(z, nthreads=2)) == e["sha256"], N


@pytest.mark.parametrize("tag,dt", [("c128", np.complex128), ("c64", np.complex64)])
def test_classical_large_digest_golden(golden, oracle_mod, tag, dt):
    _, meta = golden
    for lg in range(13, 17):
        N = 1 << lg
        e = meta["cdft_sha256"][f"classical_{tag}_{N}"]
        z = golden_input(N, e["batch"], dt, e["seed"])
        assert sha(oracle_mod.cdft(z, algo="classical", nthreads=2)) == e["sha256"], N


def real_input(n_vals, B, dt, seed):
    """Same generator as tests/golden/make_golden.py:real_input."""
    return np.random.default_rng(seed).standard_normal((n_vals, B)).astype(dt)


@pytest.mark.parametrize("algo", ["improved", "classical"])
@pytest.mark.parametrize("kind", ["rdft", "dct0", "dst0"])
@pytest.mark.parametrize("tag,dt", [("f64", np.float64), ("f32", np.float32)])
def test_real_kinds_golden(golden, oracle_mod, algo, kind, tag, dt):
    """rdft / dct0 / dst0 (improved.py:117-136, classical.py:134-153): raw
    outputs up to 2^10 and digests up to 2^16, generated by the reference."""
    arrays, meta = golden
    fn = getattr(oracle_mod, kind)
    for lg in range(1 if kind != "dst0" else 2, 17):
        N = 1 << lg
        key = f"{algo}_{kind}_{tag}_{N}"
        e = meta["real_sha256"][key]
        x = real_input(e["n_vals"], e["batch"], dt, e["seed"])
        got = fn(x, algo=algo, nthreads=2)
        if lg <= 10:
            assert bit_equal(x, arrays[f"in_{kind}_{tag}_{N}"])
            assert bit_equal(got, arrays[key]), key
        assert sha(got) == e["sha256"], key


def config_rows_input(c, meta):
    from paper_1301_0763_b200 import workloads
    e = meta["config_rows"][str(c)]
    N = e["N"]
    if c in (2, 5):
        return workloads.keyed_normal_rows(N, 2, 0, e["seed"], np.complex64)
    if c == 3:
        return workloads.config3_rows(N, 2, 0, e["seed"])
    return workloads.uniform_rows(N, 2, e["seed"], np.complex128)


@pytest.mark.parametrize("c", [2, 3, 4, 5])
def test_config_rows_golden(golden, oracle_mod, c):
    """Rows 0 and 1 of every BASELINE configuration's own input (the generators
    bench.py uses): the input digest pins the generator, the output digest is
    the reference's improved.cdft of those rows."""
    _, meta = golden
    e = meta["config_rows"][str(c)]
    x = config_rows_input(c, meta)
    assert sha(x) == e["input_sha256"]
    assert sha(oracle_mod.cdft_rows(x, nthreads=2)) == e["improved_sha256"]
    if "classical_sha256" in e:
        assert sha(oracle_mod.cdft_rows(x, algo="classical", nthreads=2)) == e["classical_sha256"]
