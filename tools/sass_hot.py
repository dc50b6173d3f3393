#!/usr/bin/env python
"""Top SASS lines by warp-stall samples from an ncu report (source page)."""
import csv
import io
import subprocess
import sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ai, si, wi = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) == len(h)]
tot = sum(int(r[wi]) for r in data)
print(f"total samples {tot}")
idx = {r[ai]: i for i, r in enumerate(data)}
for r in sorted(data, key=lambda r: -int(r[wi]))[:top]:
    print(f"{int(r[wi]):7d} {100*int(r[wi])/tot:5.1f}%  [{idx[r[ai]]:4d}] {r[si].strip()[:90]}")
