"""Per global-memory SASS instruction of an ncu report: stall samples, L1 tag
requests and L2 sectors (theoretical vs ideal), top N by samples."""
import csv, io, subprocess, sys
rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[ix[k]].replace(",", ""))
    except Exception: return 0.0
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in rows[2:]) or 1
g = [r for r in rows[2:] if "LDG" in r[ix["Source"]] or "STG" in r[ix["Source"]]]
print(f"global instructions {len(g)}: samples {100*sum(f(r,'Warp Stall Sampling (All Samples)') for r in g)/tot:.1f}%")
for r in sorted(g, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
    ex = f(r, "Instructions Executed") or 1
    print(f"{r[ix['Address']]:>6} {r[ix['Source']][:38]:38s} samp {100*f(r,'Warp Stall Sampling (All Samples)')/tot:5.2f}% exec {ex:9.0f} "
          f"tagreq/inst {f(r,'L1 Tag Requests Global')/ex:5.1f} sect/inst {f(r,'L2 Theoretical Sectors Global')/ex:5.1f} (ideal {f(r,'L2 Theoretical Sectors Global Ideal')/ex:5.1f})")
