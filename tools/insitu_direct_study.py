#!/usr/bin/env python
"""In situ execution-method study with a compute-bound producer (SURVEY.md
8(f) row 4; the paper's lockstep vs asynchronous comparison, PAPER.md:500-505,
:518-526).

Producer: an O(N^2) fp64 direct-sum gravity step (synth.direct_step; the
Newton++ solver class) on GPU 0.  Analysis after every
step: the paper's in situ step in miniature -- the fused multi-instance
DataBin over 9 coordinate systems x 7 variables at 256^2 (R19,
bin_multi_*), on the same GPU:
  lockstep        on the solver's stream
  async_snapshot  side stream, deep copy of the columns first
  async_inplace   side stream, reads in place; the solver's next drift waits
                  for bin_multi_inputs_released
Reported per mode: solver ms/step, apparent in situ ms/step (time the
solver's stream is held), actual in situ ms/step, total ms.  Checks: the
solver trajectory is bit-identical in every mode and the final step's grids
match the oracle.

  python tools/insitu_direct_study.py [--n 262144] [--steps 30]
"""
import argparse
import ctypes
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tools.placement_study import _cudart  # noqa: E402

SYSTEMS = [(0, 1), (0, 2), (1, 2), (4, 5), (4, 6), (5, 6), (0, 4), (1, 5), (2, 6)]
NAMES = ("x", "y", "z", "mass", "vx", "vy", "vz")  # column order of the instance table (R19)


def run(mode, n, steps, dt=1e-6, seed=7):
    import torch

    import paper_2310_02926_b200 as db
    import synth
    cudart = _cudart()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    S = torch.cuda.Stream(dev)
    cols = {}
    for c in NAMES:
        t = torch.empty(n, dtype=torch.float64, device=dev)
        synth.fill_device(synth.UNIFORM, 1, seed, synth.COLUMNS[c], 0, n, t.data_ptr(), S.cuda_stream)
        cols[c] = t
    torch.cuda.synchronize()
    arrs = [db.wrap_tensor(cols[c], stream=S.cuda_stream, mode=db.BIN_ASYNC) for c in NAMES]
    place = {"lockstep": db.make_placement(device_id=0, exec=db.BIN_EXEC_SYNC),
             "async_snapshot": db.make_placement(device_id=0, exec=db.BIN_EXEC_ASYNC, async_snapshot=1),
             "async_inplace": db.make_placement(device_id=0, exec=db.BIN_EXEC_ASYNC, async_snapshot=0)}[mode]
    specs = [db.make_spec((256, 256), (-4.0, -4.0), (4.0, 4.0), nattr=7) for _ in SYSTEMS]
    m = db.bin_multi_init([db.make_multi_op(sp, s, range(7)) for sp, s in zip(specs, SYSTEMS)], 7, place)
    db.bin_multi_profile_enable(m, True)
    ptrs = [cols[c].data_ptr() for c in ("x", "y", "z", "vx", "vy", "vz", "mass")]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    ev_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ticket = None
    for k in range(steps):
        ev[k][0].record(S)
        synth.direct_step(ptrs, n, S.cuda_stream, dt=dt)
        ev[k][1].record(S)
        ticket = db.bin_multi_execute(m, arrs)
        if mode != "lockstep":
            rel = db.bin_multi_inputs_released(m, ticket)
            assert cudart.cudaStreamWaitEvent(ctypes.c_void_p(S.cuda_stream), ctypes.c_void_p(rel), 0) == 0
    ev_end.record(S)
    db.bin_multi_wait(m, ticket)
    outs = [db.result_to_numpy(m, ticket, sp, op=k) for k, sp in enumerate(specs)]
    torch.cuda.synchronize()
    total_ms = (time.perf_counter() - t0) * 1e3
    prof = db.bin_multi_profile_read(m)
    solver = [ev[k][0].elapsed_time(ev[k][1]) for k in range(steps)]
    apparent = [ev[k][1].elapsed_time(ev[k + 1][0]) for k in range(steps - 1)] + [ev[-1][1].elapsed_time(ev_end)]
    actual = (prof.ms_init + prof.ms_bounds + prof.ms_bin + prof.ms_combine + prof.ms_finalize) / max(1, prof.executes)
    final = {c: cols[c].cpu().numpy() for c in NAMES}
    state = hashlib.sha256(b"".join(final[c].tobytes() for c in NAMES)).hexdigest()
    db.bin_multi_finalize(m)
    for a in arrs:
        db.bin_array_release(a)
    return ({"mode": mode, "n": n, "steps": steps, "solver_ms_per_step": sum(solver[1:]) / max(1, steps - 1),
             "apparent_insitu_ms_per_step": sum(apparent[1:]) / max(1, steps - 1),
             "actual_insitu_ms_per_step": actual, "total_ms": total_ms, "state_sha256": state[:16],
             "analysis": "fused 9 systems x 7 variables, 256^2 (bin_multi)"}, outs, final)


def check(results):
    import oracle
    from tests.gpu_util import compare
    assert len({r["state_sha256"] for r, _, _ in results}) == 1, "solver trajectories differ between modes"
    _, _, final = results[0]
    cols = [final[c] for c in NAMES]
    for _, outs, _ in results:
        for s, out in zip(SYSTEMS, outs):
            compare(out, oracle.databin([cols[s[0]], cols[s[1]]], cols, (256, 256), (-4.0, -4.0), (4.0, 4.0)))
    return True


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=262144)
    ap.add_argument("--steps", type=int, default=30)
    args = ap.parse_args()
    results = [run(mo, args.n, args.steps) for mo in ("lockstep", "async_snapshot", "async_inplace")]
    ok = check(results)
    for r, _, _ in results:
        print(json.dumps(r), flush=True)
    print(json.dumps({"parity_vs_oracle_and_modes": ok}), flush=True)


if __name__ == "__main__":
    main()
