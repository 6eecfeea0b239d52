"""Per-segment (BAR.SYNC-delimited) stall breakdown of an ncu report's SASS source page."""
import csv, io, subprocess, sys
rep = sys.argv[1]
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
keys = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
def f(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except Exception:
        return 0.0
segs = []; cur = {k: 0.0 for k in keys}; cur["n"] = 0
for r in data:
    for k in keys: cur[k] += f(r, k)
    cur["n"] += 1
    if "BAR.SYNC" in r[ix["Source"]] or "BAR.SYNC" in r[ix["Source"]].upper():
        segs.append(cur); cur = {k: 0.0 for k in keys}; cur["n"] = 0
segs.append(cur)
tot = sum(sum(s[k] for k in keys) for s in segs) or 1
for i, s in enumerate(segs):
    t = sum(s[k] for k in keys)
    top = sorted(((k, s[k]) for k in keys), key=lambda kv: -kv[1])[:6]
    print(f"seg{i} n={s['n']:5d} {100*t/tot:5.1f}% | " + " ".join(f"{k[6:]}:{100*v/tot:.1f}" for k, v in top))
