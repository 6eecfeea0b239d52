"""Summarise an ncu report of the smem kernel: headline metrics, stall reasons,
per-phase (BAR.SYNC-delimited) instruction / smem-wavefront breakdown."""
import csv, io, subprocess, sys
rep = sys.argv[1]
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
          "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
          "smsp__thread_inst_executed_per_inst_executed.ratio"]:
    if k in d:
        print(f"{k:60s} {d[k]}")
st = [(k, float(v.replace(",", "") or 0)) for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
tot = sum(v for _, v in st) or 1
print("stalls: " + ", ".join(f"{k[33:]} {100*v/tot:.1f}%" for k, v in sorted(st, key=lambda kv: -kv[1])[:8]))
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except Exception:
        return 0.0
seg = []; cur = {"n": 0, "samp": 0, "inst": 0, "wf": 0, "wfi": 0, "ops": {}}
for r in data:
    src = r[ix["Source"]]
    cur["n"] += 1; cur["samp"] += f(r, "Warp Stall Sampling (All Samples)"); cur["inst"] += f(r, "Instructions Executed")
    cur["wf"] += f(r, "L1 Wavefronts Shared"); cur["wfi"] += f(r, "L1 Wavefronts Shared Ideal")
    toks = src.split()
    op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")
    op = op.split(".")[0]
    cur["ops"][op] = cur["ops"].get(op, 0) + f(r, "Instructions Executed")
    if "BAR.SYNC" in src:
        seg.append(cur); cur = {"n": 0, "samp": 0, "inst": 0, "wf": 0, "wfi": 0, "ops": {}}
seg.append(cur)
tot = sum(s["samp"] for s in seg) or 1; ti = sum(s["inst"] for s in seg) or 1
print(f"SASS instructions {sum(s['n'] for s in seg)}, warp-instructions per transform {ti/batch:.0f}")
for i, s in enumerate(seg):
    top = sorted(s["ops"].items(), key=lambda kv: -kv[1])[:7]
    print(f"seg{i} n={s['n']:5d} samples {100*s['samp']/tot:5.1f}% inst {100*s['inst']/ti:5.1f}% smem wf/tr {s['wf']/batch:5.0f} (ideal {s['wfi']/batch:5.0f}) | "
          + " ".join(f"{k}:{v/batch:.0f}" for k, v in top))
