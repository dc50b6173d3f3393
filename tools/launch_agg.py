#!/usr/bin/env python
"""Aggregate an ncu launch list (--csv --metrics gpu__time_duration.sum,dram__bytes_*) over the
last execute (from the last launch whose name contains MARK, default k_prep)."""
import collections
import csv
import sys

path = sys.argv[1]
mark = sys.argv[2] if len(sys.argv) > 2 else "k_prep"
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    per.setdefault(r[ii], {"k": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
items = list(per.values())
idx = [i for i, it in enumerate(items) if mark in it["k"]]
last = items[idx[-1]:] if idx else items
agg = collections.OrderedDict()
for it in last:
    k = it["k"].split("(")[0].replace("void ", "")
    a = agg.setdefault(k, [0.0, 0, 0.0])
    a[0] += it.get("gpu__time_duration.sum", 0) / 1e3
    a[1] += 1
    a[2] += (it.get("dram__bytes_read.sum", 0) + it.get("dram__bytes_write.sum", 0)) / 1e6
tot = sum(a[0] for a in agg.values())
for k, a in agg.items():
    print(f"{k:44s} {a[0]:9.1f} us  x{a[1]:<3d} {a[2]:9.0f} MB")
print(f"{'total':44s} {tot:9.1f} us")
