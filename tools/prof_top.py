"""Top SASS instructions of an ncu report by stall samples, with the dominant stall reasons."""
import csv, io, subprocess, sys
rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[ix[k]].replace(",", ""))
    except Exception: return 0.0
data = rows[2:]
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for n, r in sorted(enumerate(data), key=lambda nr: -f(nr[1], "Warp Stall Sampling (All Samples)"))[:top]:
    s = f(r, "Warp Stall Sampling (All Samples)")
    rs = sorted(((h[6:], f(r, h)) for h in st), key=lambda kv: -kv[1])[:3]
    print(f"#{n:5d} {100*s/tot:5.2f}% {r[ix['Source']][:44]:44s} " + " ".join(f"{k}:{100*v/max(s,1):.0f}%" for k, v in rs))
