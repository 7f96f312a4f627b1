"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv): per kernel count/mean/min/max."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hi], rows[hi + 1:]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = collections.defaultdict(list)
for r in data:
    if len(r) > vi:
        d[r[ki][:48]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in d.values())
for k, v in d.items():
    print(f"{k:48s} n={len(v):4d} mean={sum(v)/len(v)/1e3:8.2f}us min={min(v)/1e3:8.2f} "
          f"max={max(v)/1e3:8.2f} share={sum(v)/tot:6.1%}")
