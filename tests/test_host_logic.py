"""Host-side logic of the drop-in: counter semantics, constant tables and the
TrigTable access log, against fixtures produced by the reference."""

import numpy as np
import pytest

from paper_1301_0763_b200.counting import (OpCounter, TrigTable, build_trig_table,
                                           improved_cdft_counts, natural_constants)


def test_closed_form_matches_reference_counts(golden):
    _, meta = golden
    for N, (adds, muls) in meta["cdft_counts"].items():
        assert improved_cdft_counts(int(N)) == (adds, muls)
    for N, (adds, muls) in meta["cdft_counts_batch2"].items():
        a, m = improved_cdft_counts(int(N))
        assert (2 * a, 2 * m) == (adds, muls)


@pytest.mark.parametrize("tag,dt", [("f64", np.float64), ("f32", np.float32)])
def test_trigtable_values_bitwise(golden, tag, dt):
    arrays, _ = golden
    for lg in range(3, 13):
        N = 1 << lg
        t = TrigTable(dtype=dt)
        got = natural_constants(t, N)
        assert got.tobytes() == arrays[f"table_{tag}_{N}"].tobytes(), N


def test_single_tier_values(golden):
    arrays, _ = golden
    t = TrigTable(dtype=np.float64, pipeline="single_tier")
    assert natural_constants(t, 4096).tobytes() == arrays["table_f64_single_4096"].tobytes()


def test_touched_footprint_keys(golden):
    _, meta = golden
    t = build_trig_table("improved", 64, np.float64)
    assert t.touched_count() == 0
    natural_constants(t, 64)
    want = {tuple(k) for k in meta["touched_64"]}
    assert t.touched == want
    assert t.touched_count() == 64 // 4


def test_opcounter():
    c = OpCounter()
    c.adds += 3
    c.muls += 2
    assert c.flops == 5
    c.reset()
    assert (c.adds, c.muls) == (0, 0)


def test_table_errors():
    with pytest.raises(ValueError):
        TrigTable(dtype=np.int32)
    with pytest.raises(ValueError):
        TrigTable(pipeline="x")
    with pytest.raises(ValueError):
        TrigTable().half_secant(4, 16)
    with pytest.raises(ValueError):
        build_trig_table("fancy", 16)


def test_classical_counts_replay_matches_reference(golden):
    from paper_1301_0763_b200.counting import classical_counts
    _, meta = golden
    for key, (adds, muls) in meta["classical_counts"].items():
        kind, N = key.split("_")
        assert classical_counts(kind, int(N)) == (adds, muls), key
