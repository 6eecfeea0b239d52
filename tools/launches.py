"""Summarise an ncu --csv launch list: per kernel name, count and mean of each metric."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr, acc = None, defaultdict(lambda: defaultdict(list))
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        try:
            acc[d["Kernel Name"][:70]][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
        except ValueError:
            pass
for k, m in acc.items():
    print(k)
    for name, v in m.items():
        print(f"   {name:60s} n={len(v):3d} mean={sum(v) / len(v):.4g}")
