#!/usr/bin/env python
"""Fused multi-operator binning vs the paper's sequential instances (C6).

The paper's in situ step: the DataBin operator on the Newton++ variables over
9 coordinate systems, "each coordinate system ... in a separate data binning
operator instance" run sequentially.  Here the 7 synthetic
Newton++ columns (x, y, z, mass, vx, vy, vz; R19) are binned over
the 9 systems xy, xz, yz, vx-vy, vx-vz, vy-vz, x-vx, y-vy, z-vz at 256^2, each
instance reducing count + sum/min/max/avg of all 7 variables.

  fused:      one bin_multi_execute per step (3 kernel launches for all 9)
  sequential: 9 bin_execute calls per step on 9 handles (the paper's way)

Rows per step: the paper's per-rank share (24M bodies over 512 GPUs =
46,875) and larger single-GPU sizes.  CUDA events on the launch stream, W
warm-up steps, K timed steps; prints one JSON line per (rows, mode).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SYSTEMS = [(0, 1), (0, 2), (1, 2), (4, 5), (4, 6), (5, 6), (0, 4), (1, 5), (2, 6)]
NAMES = ["x", "y", "z", "mass", "vx", "vy", "vz"]
COLS = [0, 1, 2, 3, 4, 5, 6]  # synth column ids in NAMES order: x y z m vx vy vz


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rows", default="46875,1000000,24000000")
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--res", type=int, default=256)
    a = p.parse_args()
    import torch

    import paper_2310_02926_b200 as db
    import synth
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(dev)
    R = a.res
    for n in [int(x) for x in a.rows.split(",")]:
        cols = []
        for c in COLS:
            t = torch.empty(n, dtype=torch.float64, device=dev)
            synth.fill_device(synth.UNIFORM, 1, 6, c, 0, n, t.data_ptr(), stream.cuda_stream)
            cols.append(t)
        torch.cuda.synchronize()
        arrs = [db.wrap_tensor(t, stream=stream.cuda_stream, mode=db.BIN_ASYNC) for t in cols]
        specs = [db.make_spec((R, R), (-1.0, -1.0), (1.0, 1.0), nattr=7) for _ in SYSTEMS]
        place = db.make_placement(device_id=0)

        def timed(step, prof_read):
            t = None
            for _ in range(a.warmup):
                t = step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(a.steps):
                t = step()
            e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / a.steps, t

        # fused
        m = db.bin_multi_init([db.make_multi_op(sp, s, COLS) for sp, s in zip(specs, SYSTEMS)], 7, place)
        db.bin_multi_profile_enable(m, True)
        ms_f, t = timed(lambda: db.bin_multi_execute(m, arrs), None)
        db.bin_multi_wait(m, t)
        pf = db.bin_multi_profile_read(m)
        fused_counts = [db.result_to_numpy(m, t, specs[k], op=k)["count"] for k in range(len(SYSTEMS))]
        db.bin_multi_finalize(m)
        # sequential instances (the paper's orchestration)
        hs = [db.bin_init(sp, place) for sp in specs]
        for h in hs:
            db.bin_profile_enable(h, True)
        last = [None] * len(hs)

        def seq():
            for k, (h, s) in enumerate(zip(hs, SYSTEMS)):
                last[k] = db.bin_execute(h, [arrs[s[0]], arrs[s[1]]], arrs)
            return last[-1]
        ms_s, _ = timed(seq, None)
        for h, t in zip(hs, last):
            db.bin_wait(h, t)
        launches_s = sum(db.bin_profile_read(h).kernel_launches for h in hs)
        execs_s = db.bin_profile_read(hs[0]).executes
        same = all((db.result_to_numpy(h, t, specs[k])["count"] == fused_counts[k]).all()
                   for k, (h, t) in enumerate(zip(hs, last)))
        for h in hs:
            db.bin_finalize(h)
        for x in arrs:
            db.bin_array_release(x)
        alg = n * 7 * 8
        for mode, ms, launches in (("fused", ms_f, pf.kernel_launches / max(1, pf.executes)),
                                   ("sequential", ms_s, launches_s / max(1, execs_s))):
            print(json.dumps({
                "workload": "c6_paper_step_9x7_%dx%d" % (R, R), "mode": mode, "rows": n, "ms_per_step": ms,
                "rows_per_s": n / (ms * 1e-3), "bin_updates_per_s": n * 9 * 22 / (ms * 1e-3),
                "launches_per_step": launches, "alg_bytes_per_step": alg,
                "phases_ms": ({k: getattr(pf, "ms_" + k) / max(1, pf.executes)
                               for k in ("init", "bounds", "bin", "combine", "finalize")} if mode == "fused" else None),
                "counts_equal_fused_vs_sequential": bool(same)}), flush=True)
        del cols


if __name__ == "__main__":
    main()
