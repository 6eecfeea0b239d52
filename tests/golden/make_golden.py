"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
package itself (read-only at /root/reference/pkg/src).  Run in the build
container:  python tests/golden/make_golden.py

Everything here is produced by the reference's own code path
(quickfourier.improved / classical / counting / reference) or taken from the
reference's own test modules (frozen known-answer vectors), so the oracle and
the GPU path are pinned to the reference, not to a restatement of it.
"""

import hashlib
import importlib.util
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)
sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))  # the repo (workloads generators)

from quickfourier import classical, improved, reference  # noqa: E402
from quickfourier.counting import OpCounter, TrigTable, build_trig_table  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load_ref_test(name):
    spec = importlib.util.spec_from_file_location(name, os.path.join(REF_TESTS, name + ".py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def natural(N, dt):
    t = TrigTable(dtype=dt)
    return np.array([t.eighth_cos()] + [t.half_secant(m, N) for m in range(1, N // 4)], dtype=dt)


def golden_input(N, B, dt, seed):
    """Seeded input of the golden cases: re block then im block, N(0,1)."""
    rng = np.random.default_rng(seed)
    re = rng.standard_normal((N, B))
    im = rng.standard_normal((N, B))
    return (re + 1j * im).astype(dt)


def real_input(n_vals, B, dt, seed):
    """Seeded real input of the rdft / dct0 / dst0 cases: (n_vals, B), N(0,1)."""
    return np.random.default_rng(seed).standard_normal((n_vals, B)).astype(dt)


def config1_input():
    """BASELINE config 1: c128, N=2^10, batch 64, re/im i.i.d. U[-1,1) from seed 0."""
    rng = np.random.default_rng(0)
    N, B = 1 << 10, 64
    re = rng.uniform(-1.0, 1.0, (N, B))
    im = rng.uniform(-1.0, 1.0, (N, B))
    return re + 1j * im


def main():
    arrays = {}
    meta = {"generator": "tests/golden/make_golden.py", "reference": REF_SRC, "numpy": np.__version__}

    # 1. constant tables (two-tier), raw up to 4096, digests above
    meta["table_sha256"] = {}
    for dt, tag in ((np.float64, "f64"), (np.float32, "f32")):
        for lg in range(3, 21):
            N = 1 << lg
            T = natural(N, dt)
            if lg <= 12:
                arrays[f"table_{tag}_{N}"] = T
            meta["table_sha256"][f"{tag}_{N}"] = sha(T)
    # single-tier f64 (pipeline comparison of the accuracy harness)
    t = TrigTable(dtype=np.float64, pipeline="single_tier")
    arrays["table_f64_single_4096"] = np.array(
        [t.eighth_cos()] + [t.half_secant(m, 4096) for m in range(1, 1024)])

    # 2. seeded improved/classical cdft: raw for N <= 1024, digests above
    meta["cdft_sha256"] = {}
    for dt, tag in ((np.complex128, "c128"), (np.complex64, "c64")):
        for lg in range(1, 17):
            N = 1 << lg
            B = 3 if lg <= 10 else (2 if lg <= 14 else 1)
            z = golden_input(N, B, dt, 1000 + lg)
            out_i = improved.cdft(z)
            if lg <= 10:
                arrays[f"in_{tag}_{N}"] = z
                arrays[f"improved_{tag}_{N}"] = out_i
            meta["cdft_sha256"][f"improved_{tag}_{N}"] = {"seed": 1000 + lg, "batch": B, "sha256": sha(out_i)}
            if lg <= 12:
                out_c = classical.cdft(z)
                meta["cdft_sha256"][f"classical_{tag}_{N}"] = {"seed": 1000 + lg, "batch": B, "sha256": sha(out_c)}

    # 3. known-answer vectors from the reference's own tests
    tr = load_ref_test("test_reference")
    z8 = np.array(tr.RE8) + 1j * np.array(tr.IM8)
    arrays["kat_cdft8_in"] = z8
    arrays["kat_cdft8_frozen"] = np.array(tr.CDFT8_RE) + 1j * np.array(tr.CDFT8_IM)  # 50-digit values
    arrays["kat_cdft8_improved"] = improved.cdft(z8)
    arrays["kat_cdft8_improved_c64"] = improved.cdft(z8.astype(np.complex64))
    rot = np.array([1, 1j, -1, -1j])
    arrays["kat_rot4_improved"] = improved.cdft(rot)          # test_reference.py:222-225 / test_cli.py:51-60
    imp = np.zeros(16, dtype=np.complex128)
    imp[0] = 1.0
    arrays["kat_impulse16_improved"] = improved.cdft(imp)     # impulse -> all ones (test_cli.py:19-25)

    # 4. config 1 (full batch) -- digest of the reference's output
    z1 = config1_input()
    out1 = improved.cdft(z1)
    meta["config1"] = {"input_sha256": sha(z1), "improved_sha256": sha(out1),
                       "classical_sha256": sha(classical.cdft(z1))}

    # 5. op counts and constant footprint (test_improved.py:10-21, :127-145)
    ti = load_ref_test("test_improved")
    meta["cdft_counts"] = {str(k): list(v) for k, v in ti.CDFT_COUNTS.items()}
    counts = {}
    for lg in range(1, 13):
        N = 1 << lg
        c = OpCounter()
        improved.cdft(golden_input(N, 2, np.complex128, 7), counter=c)
        counts[str(N)] = [c.adds, c.muls]
    meta["cdft_counts_batch2"] = counts
    ccounts = {}
    for lg in range(1, 13):
        N = 1 << lg
        for kind in ("cdft", "rdft", "dct0", "dst0"):
            if kind == "dst0" and N < 4:
                continue
            n_vals = {"cdft": N, "rdft": N, "dct0": N // 2 + 1, "dst0": N // 2 - 1}[kind]
            x = np.random.default_rng(1).uniform(-0.5, 0.5, n_vals)
            if kind == "cdft":
                x = x + 1j * x
            c = OpCounter()
            getattr(classical, kind)(x, counter=c)
            ccounts[f"{kind}_{N}"] = [c.adds, c.muls]
    meta["classical_counts"] = ccounts
    table = build_trig_table("improved", 64, np.float64)
    improved.cdft(golden_input(64, 1, np.complex128, 1)[:, 0], table=table, counter=OpCounter())
    meta["touched_64"] = sorted([list(k) for k in table.touched])

    # 6. large improved cdft (2^17 .. 2^20) and classical cdft up to 2^16: digests
    for dt, tag in ((np.complex128, "c128"), (np.complex64, "c64")):
        for lg in range(17, 21):
            N = 1 << lg
            B = 2 if lg <= 18 else 1
            z = golden_input(N, B, dt, 1000 + lg)
            meta["cdft_sha256"][f"improved_{tag}_{N}"] = {"seed": 1000 + lg, "batch": B,
                                                          "sha256": sha(improved.cdft(z))}
        for lg in range(13, 17):
            N = 1 << lg
            B = 2 if lg <= 14 else 1
            z = golden_input(N, B, dt, 1000 + lg)
            meta["cdft_sha256"][f"classical_{tag}_{N}"] = {"seed": 1000 + lg, "batch": B,
                                                           "sha256": sha(classical.cdft(z))}

    # 7. real-input entry points rdft / dct0 / dst0 (improved.py:117-136,
    #    classical.py:134-153): raw outputs up to 2^10, digests up to 2^16
    meta["real_sha256"] = {}
    for dt, tag in ((np.float64, "f64"), (np.float32, "f32")):
        for kind in ("rdft", "dct0", "dst0"):
            for lg in range(1 if kind != "dst0" else 2, 17):
                N = 1 << lg
                n_vals = {"rdft": N, "dct0": N // 2 + 1, "dst0": N // 2 - 1}[kind]
                B = 3 if lg <= 10 else (2 if lg <= 14 else 1)
                x = real_input(n_vals, B, dt, 2000 + lg)
                for algo, mod in (("improved", improved), ("classical", classical)):
                    y = getattr(mod, kind)(x)
                    key = f"{algo}_{kind}_{tag}_{N}"
                    if lg <= 10:
                        arrays[f"in_{kind}_{tag}_{N}"] = x
                        arrays[key] = y
                    meta["real_sha256"][key] = {"seed": 2000 + lg, "batch": B, "n_vals": n_vals, "sha256": sha(y)}

    # 8. the BASELINE configurations' own inputs (rows 0 and 1 of each, from the
    #    generators bench.py and the -m gpu tests use): input and reference-output
    #    digests, batch-major rows transformed as (N, 2) columns
    from paper_1301_0763_b200 import workloads
    meta["config_rows"] = {}
    rows = {
        2: workloads.keyed_normal_rows(1 << 12, 2, 0, workloads.SEEDS[2], np.complex64),
        3: workloads.config3_rows(1 << 16, 2, 0, workloads.SEEDS[3]),
        4: workloads.uniform_rows(1 << 20, 2, workloads.SEEDS[4], np.complex128),
        5: workloads.keyed_normal_rows(1 << 14, 2, 0, workloads.SEEDS[5], np.complex64),
    }
    for c, x in rows.items():
        y = improved.cdft(np.ascontiguousarray(x.T)).T
        meta["config_rows"][str(c)] = {"N": int(x.shape[1]), "rows": [0, 1], "seed": workloads.SEEDS[c],
                                       "input_sha256": sha(x), "improved_sha256": sha(np.ascontiguousarray(y))}
    meta["config_rows"]["4"]["classical_sha256"] = sha(np.ascontiguousarray(
        classical.cdft(np.ascontiguousarray(rows[4].T)).T))

    np.savez_compressed(os.path.join(OUT, "golden.npz"), **arrays)
    with open(os.path.join(OUT, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays;", os.path.getsize(os.path.join(OUT, "golden.npz")), "bytes")


if __name__ == "__main__":
    main()
