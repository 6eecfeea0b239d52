"""Build profiles/<round>_summary.json from a tools/final_measure.sh output
directory: per config the kernels of one step (launch list: mean cold duration
and DRAM bytes per launch), the dominant kernel and its share of the step, and
-- from the ncu --set full capture of the dominant kernel -- the pipe
utilisations that bound it (HBM, shared-memory / L1 data pipe, issue).
usage: python tools/make_summary.py gpurun_out/<tag> profiles/<round>_summary.json <round>"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

src, dst, rnd = sys.argv[1], sys.argv[2], sys.argv[3]
CFG = {2: (12, 16384, 8), 3: (16, 2048, 8), 4: (20, 64, 16), 5: (14, 1 << 18, 8)}  # log2 N, batch, bytes/cell
FULL = {2: "prof_c2", 3: "prof_c3", 4: "prof_c4", 5: "prof_c5"}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, acc, order = None, defaultdict(lambda: defaultdict(list)), []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k = d["Kernel Name"].split("(")[0]
            if k not in order:
                order.append(k)
            try:
                acc[k][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
            except ValueError:
                pass
    return order, acc


out = {"round": rnd, "source": f"tools/final_measure.sh on one B200 ({src}); launch lists: ncu --metrics "
       "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none; "
       "pipe utilisations: ncu --set full of the dominant kernel"}
for c, (lg, batch, cb) in CFG.items():
    p = os.path.join(src, f"launches_c{c}.csv")
    if not os.path.exists(p):
        continue
    order, acc = launches(p)
    # launches per step: the list holds (warmup + steps) = 3 steps of the same kernels
    ks = []
    for k in order:
        if "fill" in k:  # input generator (runs once before the timed steps), not part of a step
            continue
        t = acc[k]["gpu__time_duration.sum"]
        n = len(t) // 3 or 1
        ks.append({"kernel": k, "launches": n, "us_cold": round(sum(t) / len(t) / 1e3, 1),
                   "dram_bytes": int(sum(acc[k]["dram__bytes_read.sum"]) / len(t) + sum(acc[k]["dram__bytes_write.sum"]) / len(t))})
    tot = sum(k["us_cold"] * k["launches"] for k in ks)
    dom = max(ks, key=lambda k: k["us_cold"] * k["launches"])
    d = {"kernels_per_step": ks, "dominant_kernel": dom["kernel"],
         "dominant_share_of_step": round(dom["us_cold"] * dom["launches"] / tot, 3),
         "traffic_bytes_per_launch": sum(k["dram_bytes"] * k["launches"] for k in ks),
         "algorithmic_bytes_per_launch": 2 * cb * (1 << lg) * batch,
         "launch_list": f"profiles/{rnd}_config{c}_launches.csv"}
    rep = os.path.join(src, FULL.get(c, "-") + ".ncu-rep")
    if os.path.exists(rep):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        m = dict(zip(rows[0], rows[2]))
        d["full_capture"] = {k: float(m[k].replace(",", "")) for k in KEYS if k in m and m[k]}
        d["full_capture"]["kernel"] = m.get("Kernel Name", "")
    out[f"config{c}"] = d
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1)[:3000])
