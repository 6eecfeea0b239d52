"""The arithmetic contract at the instruction level: the transform kernels must
contain no fused multiply-add of any width (FFMA, FFMA2, DFMA, HFMA2), so every
value is one IEEE-rounded add/sub/mul as in the reference's counted primitives
(counting.py:40-81).  Also checks the kernels really are sm_100a code and that
the fp32 path uses the packed FADD2 pipe.  CPU only (cuobjdump)."""

import functools
import os
import re
import shutil
import subprocess

import pytest

from conftest import ROOT

LIB = os.path.join(ROOT, "paper_1301_0763_b200", "libqftb200.so")


@functools.lru_cache(maxsize=1)
def sass_by_function():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "-sass", LIB], capture_output=True, text=True).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur:
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)([^;]*);", line)
            if m:
                addr, op, args = int(m.group(1), 16), m.group(3), m.group(4)
                # "HFMA2 Rd, -RZ, RZ, imm, imm" is ptxas's idiom for loading a constant
                if op.startswith("HFMA2") and "-RZ, RZ" in args:
                    op = "MOV(HFMA2-imm)"
                funcs[cur].append((op, args, addr))
    return funcs, out


def test_no_fused_multiply_add_in_transform_kernels():
    """No scalar FFMA/DFMA/HFMA2 at all.  FFMA2 is allowed only as the packed
    multiply x*c + z whose addend z is the opaque (-0,-0) pair: every register
    feeding an FFMA2 addend must be written only by loads/moves (never by
    arithmetic), so no product is ever fused into a sum."""
    funcs, _ = sass_by_function()
    kernels = {k: v for k, v in funcs.items() if "qft_cdft" in k or "lg_" in k or "cl_" in k or "classical_kernel" in k}
    assert any("cl_tree_kernel" in k for k in kernels) and any("cl_glevel_kernel" in k for k in kernels)
    assert len(kernels) >= 20, "expected the per-size transform kernels"
    for name, ops in kernels.items():
        fused = [o for o, _, _ in ops if re.match(r"(FFMA(?!2)|DFMA|HFMA)", o)]
        assert not fused, f"{name}: fused multiply-add {set(fused)} would change rounding"
        ok_src = {"LDG", "LDC", "LDCU", "ULDC", "MOV", "UMOV", "LDS", "IMAD", "LDL", "R2UR"}
        # basic-block starts: branch targets and instructions after a branch
        starts = set()
        for k, (o, a, addr) in enumerate(ops):
            if o.startswith(("BRA", "EXIT", "RET", "JMP", "BSYNC", "WARPSYNC", "CALL")):
                tgt = re.search(r"0x([0-9a-f]+)", a)
                if tgt:
                    starts.add(int(tgt.group(1), 16))
                if k + 1 < len(ops):
                    starts.add(ops[k + 1][2])
        for i, (o, args, addr) in enumerate(ops):
            if not o.startswith("FFMA2"):
                continue
            addend = re.findall(r"(U?R\d+)", args)[-1]
            # nearest earlier definition of the addend inside the same basic block
            src = None
            for o2, a2, ad2 in reversed(ops[:i]):
                m = re.match(r"\s*(U?R\d+)", a2)
                if m and m.group(1) == addend:
                    src = o2.split(".")[0]
                    break
                if ad2 in starts:
                    break
            assert src is None or src in ok_src, f"{name}: FFMA2 addend {addend} defined by {src}"


def test_sm100a_and_packed_fp32():
    funcs, out = sass_by_function()
    assert "sm_100a" in out
    # the fp32 N=4096 cdft path is the pipelined kernel (qft_pipe.cuh); the real
    # modes keep qft_cdft_smem
    for pat in ("qft_cdft_pipeILi12EfE", "qft_cdft_smemILi12EfLi1E", "qft_cdft_smemILi14EfLi0E"):
        ks = [k for k in funcs if pat in k]
        assert ks, f"{pat} kernel missing"
        ops = funcs[ks[0]]
        assert any(o.startswith("FADD2") for o, _, _ in ops), f"{pat}: fp32 adds should use the packed FADD2 pipe"
    pipe = [k for k in funcs if "qft_cdft_pipeILi12EfE" in k][0]
    ops = [o for o, _, _ in funcs[pipe]]
    assert any(o.startswith("UBLKCP") or o.startswith("UTMALDG") or "BLK" in o for o in ops), \
        "the pipelined kernel should issue TMA bulk copies"


def test_multipass_fp64_items_use_tensor_map_tma():
    """North-star item (4): the multi-pass path moves its fp64 tiles (leaf runs
    and sub-signal ranges of W0) HBM -> shared memory with tensor-map TMA
    (cp.async.bulk.tensor -> UTMALDG) into the padded layout; the single-pass
    kernels stage raw signals with bulk TMA copies (UBLKCP)."""
    funcs, _ = sass_by_function()
    items64 = [k for k in funcs if "lg_item_kernel" in k and ("Ed" in k.split("lg_item_kernel")[1][:12])]
    assert items64, "fp64 item kernels not found"
    for k in items64:
        ops = [o for o, _, _ in funcs[k]]
        assert any(o.startswith("UTMALDG") for o in ops), f"{k}: no tensor-map TMA load"
        # the leaves' spectra leave by tensor-map TMA stores of the padded rows (round 2)
        assert any(o.startswith("UTMASTG") for o in ops), f"{k}: no tensor-map TMA store"
    # the fp64 F pass stages its first-touch gathers with cp.async (LDGSTS)
    f64 = [k for k in funcs if "lg_f_staged_kernel" in k]
    assert f64 and all(any(o.startswith("LDGSTS") for o, _, _ in funcs[k]) for k in f64)
    pipe = [k for k in funcs if "qft_cdft_pipe" in k]
    assert pipe and all(any(o.startswith("UBLKCP") for o, _, _ in funcs[k]) for k in pipe)
