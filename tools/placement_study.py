#!/usr/bin/env python
"""Placement study (BASELINE.json configs[4]; the paper's Table 1 / Figs. 3-4
experiment in miniature).

A Newton++-shaped producer (synth.kdk_step: O(N) leapfrog in the field of the
massive body) advances N bodies on GPU 0 every step; after each step the
DataBin analysis bins x-y with count + sum/min/max/avg of mass on a 512x512
mesh, placed and executed as:
  lockstep        same GPU, on the solver's stream
  async_snapshot  same GPU, side stream, deep copy of the inputs
  async_inplace   same GPU, side stream, reads in place; the solver waits for
                  bin_inputs_released before overwriting
  peer            GPU 1, inputs moved by peer copy over NVLink
Reported per mode (Fig. 4 analogues): solver ms/step, apparent in situ ms/step
(time the solver's stream is held), actual in situ ms/step (the library's
own phase times), total ms.  Checks: the final grids agree across modes and
with the oracle, and the solver trajectory is bit-identical in every mode
(the analysis never writes simulation data).

  python tools/placement_study.py [--n 50000000] [--steps 100] [--modes ...]
"""
import argparse
import ctypes
import glob
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MODES = ("lockstep", "async_snapshot", "async_inplace", "peer")


def _cudart():
    import nvidia.cuda_runtime as cr
    lib = ctypes.CDLL(sorted(glob.glob(os.path.join(list(cr.__path__)[0], "lib", "libcudart.so*")))[0])
    lib.cudaStreamWaitEvent.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint]
    return lib


def run_mode(mode, n, steps, res=(512, 512), lo=(-1.0, -1.0), hi=(1.0, 1.0), seed=5, dt=1e-5):
    import torch

    import paper_2310_02926_b200 as db
    import synth
    cudart = _cudart()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    S = torch.cuda.Stream(dev)
    names = ("x", "y", "z", "vx", "vy", "vz", "mass")
    cols = {}
    for c in names:
        t = torch.empty(n, dtype=torch.float64, device=dev)
        synth.fill_device(synth.UNIFORM, 1, seed, synth.COLUMNS[c], 0, n, t.data_ptr(), S.cuda_stream)
        cols[c] = t
    torch.cuda.synchronize()
    arrs = [db.wrap_tensor(cols[c], stream=S.cuda_stream, mode=db.BIN_ASYNC) for c in ("x", "y", "mass")]
    place = {
        "lockstep": db.make_placement(device_id=0, exec=db.BIN_EXEC_SYNC),
        "async_snapshot": db.make_placement(device_id=0, exec=db.BIN_EXEC_ASYNC, async_snapshot=1),
        "async_inplace": db.make_placement(device_id=0, exec=db.BIN_EXEC_ASYNC, async_snapshot=0),
        "peer": db.make_placement(device_id=1, exec=db.BIN_EXEC_PEER),
    }[mode]
    spec = db.make_spec(res, lo, hi, nattr=1)
    h = db.bin_init(spec, place)
    db.bin_profile_enable(h, True)
    ptrs = [cols[c].data_ptr() for c in ("x", "y", "z", "vx", "vy", "vz")]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    ev_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    host_in_call = 0.0
    ticket = None
    for k in range(steps):
        ev[k][0].record(S)
        synth.kdk_step(ptrs, n, S.cuda_stream, dt=dt)
        ev[k][1].record(S)
        c0 = time.perf_counter()
        ticket = db.bin_execute(h, arrs[:2], arrs[2:])
        if mode != "lockstep":  # the solver may overwrite its arrays only after release
            rel = db.bin_inputs_released(h, ticket)
            assert cudart.cudaStreamWaitEvent(ctypes.c_void_p(S.cuda_stream), ctypes.c_void_p(rel), 0) == 0
        host_in_call += time.perf_counter() - c0
    ev_end.record(S)
    out = db.result_to_numpy(h, ticket, spec)  # waits for the last analysis
    torch.cuda.synchronize()
    total_ms = (time.perf_counter() - t0) * 1e3
    prof = db.bin_profile_read(h)
    solver = [ev[k][0].elapsed_time(ev[k][1]) for k in range(steps)]
    apparent = [ev[k][1].elapsed_time(ev[k + 1][0]) for k in range(steps - 1)] + [ev[-1][1].elapsed_time(ev_end)]
    actual = (prof.ms_stage + prof.ms_init + prof.ms_bounds + prof.ms_window + prof.ms_bin + prof.ms_combine +
              prof.ms_finalize) / max(1, prof.executes)
    state = hashlib.sha256(b"".join(cols[c].cpu().numpy().tobytes() for c in names)).hexdigest()
    final = {c: cols[c].cpu().numpy() for c in ("x", "y", "mass")}
    db.bin_finalize(h)
    for a in arrs:
        db.bin_array_release(a)
    metrics = {"mode": mode, "n": n, "steps": steps, "solver_ms_per_step": sum(solver[1:]) / max(1, steps - 1),
               "apparent_insitu_ms_per_step": sum(apparent[1:]) / max(1, steps - 1),
               "actual_insitu_ms_per_step": actual, "host_ms_per_bin_execute_call": host_in_call * 1e3 / steps,
               "total_ms": total_ms, "state_sha256": state[:16]}
    return metrics, out, final


def check(results, res=(512, 512), lo=(-1.0, -1.0), hi=(1.0, 1.0)):
    """Grids agree with the oracle on the final state in every mode; the
    solver trajectory is identical in every mode."""
    import oracle
    from tests.gpu_util import compare
    states = {m["state_sha256"] for m, _, _ in results}
    assert len(states) == 1, f"solver trajectories differ between modes: {states}"
    _, _, final = results[0]
    ref = oracle.databin([final["x"], final["y"]], [final["mass"]], res, lo, hi)
    for m, out, _ in results:
        compare(out, ref)
    return True


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=50_000_000)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--modes", nargs="*", default=list(MODES))
    args = ap.parse_args()
    import torch
    modes = [m for m in args.modes if m != "peer" or torch.cuda.device_count() > 1]
    results = [run_mode(m, args.n, args.steps) for m in modes]
    ok = check(results)
    for m, _, _ in results:
        print(json.dumps(m), flush=True)
    print(json.dumps({"parity_vs_oracle_and_modes": ok, "non_interference": True}), flush=True)


if __name__ == "__main__":
    main()
