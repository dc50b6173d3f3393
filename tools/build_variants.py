#!/usr/bin/env python
"""Build A/B variants of libdatabin.so with extra -D defines (experiments only).

    python tools/build_variants.py name=DEF1,DEF2 name2=DEF3 ...
writes paper_2310_02926_b200/variants/<name>.so (git-ignored, travels to the
GPU box); tools/gpurun/ab.sh runs bench.py against each with DATABIN_LIB."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2310_02926_b200 import build  # noqa: E402

out = os.path.join(ROOT, "paper_2310_02926_b200", "variants")
os.makedirs(out, exist_ok=True)
for arg in sys.argv[1:]:
    name, defs = arg.split("=", 1)
    path = build.build(force=True, defines=tuple(d for d in defs.split(",") if d), out=os.path.join(out, name + ".so"))
    print(name, "->", path)
