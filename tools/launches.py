"""Summarise an ncu launch-list CSV (gpu__time_duration.sum) per kernel."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
    agg.setdefault(r[ki].split("(")[0][:70], []).append(v * scale)
tot = sum(sum(v) for v in agg.values())
for k, v in agg.items():
    print(f"{k:72s} n={len(v):3d} mean={sum(v)/len(v):9.1f} us  share={sum(v)/tot:6.1%}")
