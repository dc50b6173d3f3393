#!/usr/bin/env python
"""Per-launch table from an ncu --csv --metrics launch list (last step of each kernel sequence)."""
import collections
import csv
import sys


def table(path, last=None):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        per.setdefault(r[ii], {"k": r[ki]})[r[mi]] = r[vi].replace(",", "")
    items = list(per.values())
    if last:
        items = items[-last:]
    for it in items:
        t = float(it.get("gpu__time_duration.sum", 0)) / 1e3
        rd = float(it.get("dram__bytes_read.sum", 0)) / 1e6
        wr = float(it.get("dram__bytes_write.sum", 0)) / 1e6
        red = float(it.get("lts__t_sectors_op_red.sum", 0)) / 1e6
        ws = float(it.get("lts__t_sectors_op_write.sum", 0)) / 1e6
        gbs = (rd + wr) / t if t else 0
        name = it["k"].split("(")[0].replace("void ", "")[:34]
        print(f"{name:34s} {t:10.1f} us  dram rd {rd:9.1f} MB wr {wr:9.1f} MB  {gbs:7.0f} GB/s  l2 red {red:8.2f} M  l2 wr {ws:8.2f} M")


if __name__ == "__main__":
    table(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
