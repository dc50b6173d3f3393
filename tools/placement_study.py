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
  fanin           the paper's "dedicated device" placement: the
                  N bodies are split over producer GPUs 1..G-1, each advancing its
                  shard; GPU 0 is the in situ device and bins all shards per step
                  in ONE execute (bin_execute_shards: NVLink peer copies from every
                  producer, then one accumulate + finalize)
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

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MODES = ("lockstep", "async_snapshot", "async_inplace", "peer", "fanin")


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
    state = hashlib.sha256(b"".join(cols[c].cpu().numpy().tobytes() for c in names)).hexdigest()  # column-major
    final = {c: cols[c].cpu().numpy() for c in ("x", "y", "mass")}
    db.bin_finalize(h)
    for a in arrs:
        db.bin_array_release(a)
    metrics = {"mode": mode, "n": n, "steps": steps, "solver_ms_per_step": sum(solver[1:]) / max(1, steps - 1),
               "apparent_insitu_ms_per_step": sum(apparent[1:]) / max(1, steps - 1),
               "actual_insitu_ms_per_step": actual, "host_ms_per_bin_execute_call": host_in_call * 1e3 / steps,
               "total_ms": total_ms, "state_sha256": state[:16]}
    return metrics, out, final


def run_fanin(n, steps, res=(512, 512), lo=(-1.0, -1.0), hi=(1.0, 1.0), seed=5, dt=1e-5):
    """Producers on GPUs 1..G-1 (one shard each), in situ on GPU 0 (fan-in)."""
    import torch

    import paper_2310_02926_b200 as db
    import synth
    cudart = _cudart()
    G = torch.cuda.device_count()
    P = G - 1
    names = ("x", "y", "z", "vx", "vy", "vz", "mass")
    prods = []
    for p in range(P):
        dev = torch.device("cuda", p + 1)
        r0, r1 = (p * n) // P, ((p + 1) * n) // P
        with torch.cuda.device(dev):
            S = torch.cuda.Stream(dev)
            cols = {}
            for c in names:
                t = torch.empty(r1 - r0, dtype=torch.float64, device=dev)
                synth.fill_device(synth.UNIFORM, 1, seed, synth.COLUMNS[c], r0, r1 - r0, t.data_ptr(), S.cuda_stream)
                cols[c] = t
            torch.cuda.synchronize(dev)
        arrs = [db.wrap_tensor(cols[c], stream=S.cuda_stream, mode=db.BIN_ASYNC) for c in ("x", "y", "mass")]
        prods.append(dict(dev=dev, S=S, cols=cols, n=r1 - r0, r0=r0, arrs=arrs,
                          ptrs=[cols[c].data_ptr() for c in ("x", "y", "z", "vx", "vy", "vz")], ev=[]))
    spec = db.make_spec(res, lo, hi, nattr=1)
    h = db.bin_init(spec, db.make_placement(device_id=0, exec=db.BIN_EXEC_PEER))
    db.bin_profile_enable(h, True)
    shards = [(q["arrs"][:2], q["arrs"][2:]) for q in prods]
    for q in prods:
        torch.cuda.synchronize(q["dev"])
    t0 = time.perf_counter()
    ticket = None
    for k in range(steps):
        for q in prods:
            with torch.cuda.device(q["dev"]):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(q["S"])
                synth.kdk_step(q["ptrs"], q["n"], q["S"].cuda_stream, dt=dt, start=q["r0"])
                e1.record(q["S"])
                q["ev"].append((e0, e1))
        ticket = db.bin_execute_shards(h, shards)
        rel = db.bin_inputs_released(h, ticket)
        for q in prods:  # each producer overwrites its arrays only after the copy left its GPU
            assert cudart.cudaStreamWaitEvent(ctypes.c_void_p(q["S"].cuda_stream), ctypes.c_void_p(rel), 0) == 0
    ends = []
    for q in prods:
        with torch.cuda.device(q["dev"]):
            e = torch.cuda.Event(enable_timing=True)
            e.record(q["S"])
            ends.append(e)
    out = db.result_to_numpy(h, ticket, spec)
    for q in prods:
        torch.cuda.synchronize(q["dev"])
    total_ms = (time.perf_counter() - t0) * 1e3
    prof = db.bin_profile_read(h)
    solver = max(sum(q["ev"][k][0].elapsed_time(q["ev"][k][1]) for k in range(1, steps)) / max(1, steps - 1)
                 for q in prods)
    apparent = max((sum(q["ev"][k][1].elapsed_time(q["ev"][k + 1][0]) for k in range(1, steps - 1))
                    + q["ev"][-1][1].elapsed_time(e)) / max(1, steps - 1) for q, e in zip(prods, ends))
    actual = (prof.ms_stage + prof.ms_init + prof.ms_bounds + prof.ms_window + prof.ms_bin + prof.ms_combine +
              prof.ms_finalize) / max(1, prof.executes)
    state = hashlib.sha256(b"".join(b"".join(q["cols"][c].cpu().numpy().tobytes() for q in prods)
                                    for c in names)).hexdigest()
    final = {c: np.concatenate([q["cols"][c].cpu().numpy() for q in prods]) for c in ("x", "y", "mass")}
    db.bin_finalize(h)
    for q in prods:
        for a in q["arrs"]:
            db.bin_array_release(a)
    metrics = {"mode": "fanin", "n": n, "steps": steps, "producers": P, "solver_ms_per_step": solver,
               "apparent_insitu_ms_per_step": apparent, "actual_insitu_ms_per_step": actual,
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
    modes = [m for m in args.modes if m not in ("peer", "fanin") or torch.cuda.device_count() > 1]
    results = [run_fanin(args.n, args.steps) if m == "fanin" else run_mode(m, args.n, args.steps) for m in modes]
    ok = check(results)
    for m, _, _ in results:
        print(json.dumps(m), flush=True)
    print(json.dumps({"parity_vs_oracle_and_modes": ok, "non_interference": True}), flush=True)


if __name__ == "__main__":
    main()
