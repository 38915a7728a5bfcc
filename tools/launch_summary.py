"""Condense an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel count/mean/total."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
h = None
agg = OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "")
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(
            d["Metric Unit"], 1.0)
        agg.setdefault(name, []).append(float(d["Metric Value"].replace(",", "")) * scale)
print(f"{'kernel':60s} {'count':>6s} {'mean_us':>12s} {'total_us':>14s}")
tot = sum(sum(v) for v in agg.values())
for k, v in agg.items():
    print(f"{k[:60]:60s} {len(v):6d} {sum(v)/len(v):12.1f} {sum(v):14.1f}  {100*sum(v)/tot:5.1f}%")
