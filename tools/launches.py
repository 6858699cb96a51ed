"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
t = OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) > vi:
        t.setdefault(r[ki][:70], []).append(float(r[vi].replace(",", "")))
for k, v in t.items():
    print(f"{k:70s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:8.2f} us")
