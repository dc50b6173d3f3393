#!/usr/bin/env python
"""One summary line per bench JSON file (the last JSON line in it)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads([ln for ln in open(f) if ln.startswith("{")][-1])
        print(f, d["config"]["workload"], round(d["value"] / 1e9, 2), "G/s", round(d["ms_per_step"], 4), "ms/step",
              "frac", round(d["roofline"]["frac"], 3), d.get("phases_ms_per_step"))
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
