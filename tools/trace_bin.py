#!/usr/bin/env python
"""k_bin_fast per-CTA phase trace (DATABIN_TRACE) at several row counts on one GPU -- diagnosis only.
EXACT=1: the BIN_SUM_EXACT instantiation."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DATABIN_TRACE"] = "1"


def main():
    import torch

    import paper_2310_02926_b200 as db
    import synth
    w = synth.CONFIGS["c3"]
    for n in (100_000_000, 25_000_000, 12_500_000):
        cols = []
        for c in list(w.axes) + list(w.attrs):
            t = torch.empty(n, dtype=torch.float64, device="cuda")
            synth.fill_device(w.dist, w.central, w.seed, synth.COLUMNS[c], 0, n, t.data_ptr(), 0)
            cols.append(t)
        torch.cuda.synchronize()
        exact = os.environ.get("EXACT") == "1"
        h = db.bin_init(db.make_spec(w.res, w.lo, w.hi, nattr=1, exact=exact), db.make_placement())
        hs = [db.wrap_tensor(t) for t in cols]
        print(f"--- n = {n:,}", file=sys.stderr, flush=True)
        for it in range(6):
            t = db.bin_execute(h, hs[:2], hs[2:])
            db.bin_wait(h, t)
        db.bin_finalize(h)
        for a in hs:
            db.bin_array_release(a)
        del cols
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
