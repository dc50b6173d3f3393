#!/usr/bin/env python
"""Experiment: a workload's single-instance step on the library's routes vs the
same instance run as a one-instance fused multi-operator set (L2 reductions
with min/max filter lines).  CUDA events, W warm-up, K timed steps."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2310_02926_b200 as db
    import synth
    names = sys.argv[1:] or ["c2", "c5"]
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    st = torch.cuda.Stream(dev)
    K, W = 20, 3
    for name in names:
        w = synth.CONFIGS[name]
        cols = []
        for c in w.axes + w.attrs:
            t = torch.empty(w.n, dtype=torch.float64, device=dev)
            synth.fill_device(w.dist, w.central, w.seed, synth.COLUMNS[c], 0, w.n, t.data_ptr(), st.cuda_stream)
            cols.append(t)
        torch.cuda.synchronize()
        arrs = [db.wrap_tensor(t, stream=st.cuda_stream, mode=db.BIN_ASYNC) for t in cols]
        D = len(w.axes)
        place = db.make_placement(device_id=0)

        def timed(step):
            for _ in range(W):
                step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(K):
                step()
            e1.record(st)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / K

        out = {"workload": w.name}
        for route, rname in ((db.BIN_ROUTE_AUTO, "auto"), (db.BIN_ROUTE_WINDOW, "window"),
                             (db.BIN_ROUTE_PARTITION, "partition")):
            sp = db.make_spec(w.res, w.lo, w.hi, nattr=len(w.attrs), route=route)
            h = db.bin_init(sp, place)
            out[rname] = timed(lambda: db.bin_execute(h, arrs[:D], arrs[D:]))
            db.bin_finalize(h)
        sp = db.make_spec(w.res, w.lo, w.hi, nattr=len(w.attrs))
        m = db.bin_multi_init([db.make_multi_op(sp, tuple(range(D)), tuple(range(D, len(cols))))], len(cols), place)
        out["multi1"] = timed(lambda: db.bin_multi_execute(m, arrs))
        db.bin_multi_finalize(m)
        print(json.dumps(out), flush=True)
        for a in arrs:
            db.bin_array_release(a)


if __name__ == "__main__":
    main()
