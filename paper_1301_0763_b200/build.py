"""In-tree build of libqftb200.so (sm_100a) -- ``python -m paper_1301_0763_b200.build``.

Every (precision, N) kernel instance is its own translation unit so the build
parallelises; objects are cached by source hash under build/.  Flags:
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false`` (no FMA
contraction: the kernels must reproduce the reference's one-rounding-per-op
arithmetic, counting.py:40-81).
"""

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build", "native")
LIB = os.path.join(HERE, "libqftb200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-Xptxas", "-v", "--expt-relaxed-constexpr"]
PRECS = (32, 64)
LOG2NS = range(1, 15)


def nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _headers_digest():
    h = hashlib.sha256()
    for d in (CSRC, os.path.join(ROOT, "include")):
        for f in sorted(os.listdir(d)):
            if f.endswith((".cuh", ".h", ".cu")):
                with open(os.path.join(d, f), "rb") as fh:
                    h.update(f.encode() + fh.read())
    h.update(" ".join(NVFLAGS).encode())
    return h.hexdigest()[:16]


def _compile(src, obj, defines):
    cmd = [nvcc()] + NVFLAGS + [f"-D{d}" for d in defines] + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = obj + ".log"
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src} {defines}:\n{r.stderr[-4000:]}")
    return obj


def build(jobs=None, verbose=True, defines=(), lib=None, only=None):
    """Compile all translation units (cached) and link libqftb200.so.
    ``defines``/``lib``: build an experimental variant (e.g. QFT_CTAS_PER_SM=3);
    ``only``: instance tags ("32_12", ...) that get the defines -- every other
    translation unit is the default build's object."""
    os.makedirs(BUILD, exist_ok=True)
    dig0 = _headers_digest()
    dig = dig0 + ("_" + hashlib.sha256(" ".join(defines).encode()).hexdigest()[:8] if defines else "")
    target = lib or LIB
    units = [(os.path.join(CSRC, "qft_capi.cu"), os.path.join(BUILD, f"capi_{dig}.o"), list(defines))]
    for p in PRECS:
        units.append((os.path.join(CSRC, "qft_large.cu"), os.path.join(BUILD, f"large_{p}_{dig}.o"),
                      [f"QFT_LARGE_PREC={p}"] + list(defines)))
        units.append((os.path.join(CSRC, "qft_classical.cu"), os.path.join(BUILD, f"classical_{p}_{dig}.o"),
                      [f"QFT_CL_PREC={p}"] + list(defines)))
    for p in PRECS:
        for l in LOG2NS:
            d = dig if only is None or f"{p}_{l}" in only else dig0
            units.append((os.path.join(CSRC, "qft_inst.cu"), os.path.join(BUILD, f"inst_{p}_{l}_{d}.o"),
                          [f"QFT_INST_PREC={p}", f"QFT_INST_LOG2N={l}"] + (list(defines) if d == dig else [])))
    if only is not None:  # the shared units stay the default build's
        units = [(u[0], u[1].replace(dig, dig0), [x for x in u[2] if x not in defines]) if "inst_" not in u[1] else u
                 for u in units]
    todo = [u for u in units if not os.path.exists(u[1])]
    if todo:
        jobs = jobs or max(2, os.cpu_count() or 2)
        if verbose:
            print(f"[build] compiling {len(todo)} translation units with {jobs} jobs", flush=True)
        with cf.ThreadPoolExecutor(jobs) as ex:
            list(ex.map(lambda u: _compile(*u), todo))
    objs = [u[1] for u in units]
    if not defines:  # drop objects of older source digests (keeps build/ small)
        keep = set(objs) | {o + ".log" for o in objs}
        for f in os.listdir(BUILD):
            full = os.path.join(BUILD, f)
            if full not in keep and ("_" + dig.split("_")[0]) not in f and f.endswith((".o", ".o.log")):
                try:
                    os.remove(full)
                except OSError:
                    pass
    tmp = target + ".tmp"
    cmd = [nvcc()] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart"]
    subprocess.check_call(cmd)
    os.replace(tmp, target)
    if verbose:
        print(f"[build] {target}", flush=True)
    return target


def ptxas_report():
    """(kernel, registers, spill bytes) from the cached build logs."""
    import re
    rows = []
    dig = _headers_digest()
    for f in sorted(os.listdir(BUILD)):
        if not f.endswith(f"_{dig}.o.log"):
            continue
        fn = None
        for line in open(os.path.join(BUILD, f)):
            m = re.search(r"Compiling entry function '(\S+)'", line)
            if m:
                fn = m.group(1)
            m = re.search(r"(\d+) bytes spill stores", line)
            if m and fn:
                spill = int(m.group(1))
            m = re.search(r"Used (\d+) registers", line)
            if m and fn:
                rows.append((fn, int(m.group(1)), spill))
    return rows


if __name__ == "__main__":
    # python -m paper_1301_0763_b200.build [out.so DEFINE=VAL ...]
    # QFT_ONLY=32_12,32_14 restricts the defines to those instances
    if len(sys.argv) > 1:
        only = os.environ.get("QFT_ONLY")
        build(lib=os.path.abspath(sys.argv[1]), defines=tuple(sys.argv[2:]), only=only.split(",") if only else None)
    else:
        build()
