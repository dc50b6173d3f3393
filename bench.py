#!/usr/bin/env python
"""Benchmark of the in situ DataBin hot path (arXiv 2310.02926, Sec. 4.2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c3|c2|c4|c5] [--scaling strong|weak] [--deterministic]

Workload (default): BASELINE.json configs[2] -- 100M Plummer-clustered
particles binned onto a 512x512 x-y mesh, count + sum/min/max/avg of mass,
sharded across N GPUs (contiguous row blocks); the bin arrays are combined
over NVLink peer memory by one fused combine + finalize kernel (NCCL as the
fallback).  One "step" = one bin_execute over the rank's shard: accumulator
init, bin kernel(s), cross-rank combine, finalize.  Inputs are
generated on the device by the seeded generator (synth/) before timing and
are larger than L2 (2.4 GB vs 126 MB), so no L2 flush is needed.

Prints ONE JSON line (rank 0).  For N > 1 launch with torchrun; timings are
CUDA events on the launch stream, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep stdout to the one JSON line

METRIC = "particles binned/sec at 1/2/4/8 B200; achieved HBM GB/s as % of peak"
UNIT = "particles/s"
NOMINAL_HBM_GBS = 8000.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", default="c3")
    p.add_argument("--scaling", choices=["strong", "weak"], default="strong")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-numa", action="store_true", help="do not bind to the GPU's NUMA node (pinned staging pages)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--bounds-auto", action="store_true")
    p.add_argument("--deterministic", action="store_true")
    p.add_argument("--exact", action="store_true", help="BIN_SUM_EXACT: correctly rounded exact sums (R20)")
    p.add_argument("--rows", type=int, default=0, help="experiments only: override the workload's total rows")
    p.add_argument("--no-phase-events", action="store_true",
                   help="experiment: no per-phase CUDA events inside the timed region (no roofline / phase times)")
    p.add_argument("--evolve", action="store_true",
                   help="experiment: the inputs change every step (a KDK drift of every row on the bench stream "
                        "before each execute); value = rows / the library's own per-execute device time")
    p.add_argument("--ops", default="", help="experiments only: comma list of ops instead of the workload's "
                                             "('none' = count only)")
    return p.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def shard(n, rank, world):
    return (rank * n) // world, ((rank + 1) * n) // world


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def load_traffic(workload):
    """dram bytes per bin-kernel launch from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        return t.get(workload)
    except Exception:
        return None


class ClockSampler:
    """Samples SM clocks and throttle reasons via NVML during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.stop = threading.Event()
        self.ok = False
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            self.t = threading.Thread(target=self.run, daemon=True)
            self.t.start()
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        return self

    def run(self):
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
            0x80: "hw_power_brake_slowdown",
        }
        while not self.stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.0005)

    def __exit__(self, *a):
        self.stop.set()
        if self.ok:
            self.t.join(timeout=1)

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(w, seconds, rank_rows=None):
    """The oracle as it stands on a bounded sample of the workload: single-
    threaded (oracle_databin, P = 1) and in its partition mode with one block
    per host core (oracle.databin_blocks, P = nproc worker threads; the rank
    decomposition of PAPER.md:479 run on CPU cores).  ``value`` is the
    all-core rate; ``single_thread`` the sequential loop's."""
    import numpy as np

    import oracle
    import synth
    oracle.build()

    def cols(s, c, threads=0):
        return ([synth.fill_host(w.dist, w.central, w.seed, synth.COLUMNS[x], s, c, threads) for x in w.axes],
                [synth.fill_host(w.dist, w.central, w.seed, synth.COLUMNS[x], s, c, threads) for x in w.attrs])

    def run(n):
        axes, attrs = cols(0, n)
        t0 = time.perf_counter()
        oracle.databin(axes, attrs, w.res, w.lo, w.hi)
        return time.perf_counter() - t0

    probe = min(w.n, 2_000_000)
    dt = run(probe)
    rate = probe / dt
    n = int(min(w.n, max(probe, rate * seconds / 2)))
    dt = run(n) if n != probe else dt
    single = {"value": n / dt, "cores": 1, "sample": f"first {n:,} rows of {w.name}, oracle_databin, {dt:.2f} s"}
    # all cores: partition mode P = nproc over a sample sized to ~seconds/2 of work
    ncores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    nm = int(min(w.n, max(n, single["value"] * ncores * seconds / 2)))
    pre = [cols(r * nm // ncores, (r + 1) * nm // ncores - r * nm // ncores) for r in range(ncores)]
    starts = [r * nm // ncores for r in range(ncores)]

    def rows(s, c):  # pre-generated blocks: the timed part is the oracle alone
        r = starts.index(s)
        return pre[r]

    t0 = time.perf_counter()
    oracle.databin_blocks(rows, nm, w.res, w.lo, w.hi, len(w.attrs), P=ncores, chunk=1 << 62)
    dtm = time.perf_counter() - t0
    del np, pre
    return {"value": nm / dtm, "unit": UNIT, "cores": ncores, "kind": "oracle", "model": cpu_model(),
            "nproc": os.cpu_count(),
            "sample": f"first {nm:,} rows of {w.name} (seeded generator, pre-generated), oracle partition mode "
                      f"P = {ncores} (one block and worker thread per core, grids folded in rank order), "
                      f"{dtm:.2f} s",
            "single_thread": single}


def reference_arm(args):
    """--impl reference: the oracle (this tier's reference), timed on the host
    cores: its partition mode with one block and worker thread per core
    (oracle.databin_blocks, P = cores) on a bounded sample per step."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import synth
    w = synth.CONFIGS[args.workload]
    import oracle
    oracle.build()
    per_step = max(0.25, args.cpu_seconds / max(1, args.steps + args.warmup))  # K+W steps in ~a minute
    ncores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)

    def cols(s, c):
        return ([synth.fill_host(w.dist, w.central, w.seed, synth.COLUMNS[x], s, c) for x in w.axes],
                [synth.fill_host(w.dist, w.central, w.seed, synth.COLUMNS[x], s, c) for x in w.attrs])

    probe_n = min(w.n, 1_000_000)
    pax, pat = cols(0, probe_n)
    t0 = time.perf_counter()
    oracle.databin(pax, pat, w.res, w.lo, w.hi)
    rate1 = probe_n / (time.perf_counter() - t0)
    n = max(100_000, min(int(rate1 * ncores * per_step), w.n))
    starts = [r * n // ncores for r in range(ncores)]
    pre = [cols(starts[r], (r + 1) * n // ncores - starts[r]) for r in range(ncores)]

    def rows(s, c):
        return pre[starts.index(s)]

    def step():
        oracle.databin_blocks(rows, n, w.res, w.lo, w.hi, len(w.attrs), P=ncores, chunk=1 << 62)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / max(1, args.steps)
    v = n / dt
    sample = (f"first {n:,} rows of {w.name} per step (pre-generated), C oracle in partition mode P = {ncores} "
              f"(one block and worker thread per core)")
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": w.name, "rows_per_step": n, "res": list(w.res), "attrs": list(w.attrs),
                       "ops": list(w.ops)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": ncores, "kind": "oracle", "model": cpu_model(),
                             "sample": sample, "single_thread_probe": rate1},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    rank, world, local = dist_env()
    # before torch creates threads or pinned pages: the e2e leg's pinned columns land on the GPU's socket
    from paper_2310_02926_b200.numa import bind_to_gpu
    numa_node = -1 if args.no_numa else bind_to_gpu(local)
    import torch
    import torch.distributed as dist

    import paper_2310_02926_b200 as db
    import synth

    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    w = synth.CONFIGS[args.workload]
    if args.ops:
        import dataclasses
        w = dataclasses.replace(w, ops=tuple(o for o in args.ops.split(",") if o != "none"),
                                attrs=w.attrs if args.ops != "none" else ())
    N_total = (args.rows or w.n) * (world if args.scaling == "weak" else 1)
    r0, r1 = shard(N_total, rank, world)
    n = r1 - r0
    stream = torch.cuda.Stream(dev)

    # ---- inputs: generated on this GPU for rows [r0, r1) (same bits as the host generator)
    cols = {}
    for c in list(w.axes) + list(w.attrs):
        t = torch.empty(n, dtype=torch.float64, device=dev)
        synth.fill_device(w.dist, w.central, w.seed, synth.COLUMNS[c], r0, n, t.data_ptr(), stream.cuda_stream)
        cols[c] = t
    torch.cuda.synchronize(dev)

    nccl_id = None
    if world > 1:
        obj = [db.bin_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    spec = db.make_spec(w.res, w.lo, w.hi, nattr=len(w.attrs), ops=w.ops, bounds_auto=args.bounds_auto,
                        deterministic=args.deterministic, exact=args.exact)
    place = db.make_placement(device_id=db.BIN_DEVICE_AUTO)  # Eq. (1): rank -> device
    h = db.bin_init(spec, place, rank=rank, nranks=world, nccl_id=nccl_id)
    arrs = [db.wrap_tensor(cols[c], stream=stream.cuda_stream, mode=db.BIN_ASYNC) for c in list(w.axes) + list(w.attrs)]
    D = len(w.axes)

    evolve_cols = None
    if args.evolve:  # x, y (+ z, vx, vy, vz) drifted on the bench stream before every execute
        extra = {}
        for c in ("x", "y", "z", "vx", "vy", "vz"):
            if c not in cols:
                t = torch.empty(n, dtype=torch.float64, device=dev)
                synth.fill_device(w.dist, w.central, w.seed, synth.COLUMNS[c], r0, n, t.data_ptr(), stream.cuda_stream)
                extra[c] = t
        torch.cuda.synchronize(dev)
        allc = {**cols, **extra}
        evolve_cols = [allc[c].data_ptr() for c in ("x", "y", "z", "vx", "vy", "vz")]

    def step():
        if evolve_cols:
            synth.kdk_step(evolve_cols, n, stream.cuda_stream, central_mass=0.0, dt=1e-3, start=r0)
        return db.bin_execute(h, arrs[:D], arrs[D:])

    # ---- warmup
    t = None
    for _ in range(args.warmup):
        t = step()
    if t is not None:
        db.bin_wait(h, t)
    torch.cuda.synchronize(dev)

    # ---- timed region: exactly K steps, barrier + synchronize on both sides
    db.bin_profile_enable(h, not args.no_phase_events)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            t = step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    db.bin_wait(h, t)
    ms = ev0.elapsed_time(ev1) / args.steps
    prof = db.bin_profile_read(h)
    res = db.bin_result(h, t)
    n_in, n_out = int(res.n_in), int(res.n_out)

    ms_t = torch.tensor([ms, prof.ms_bin / max(1, prof.executes)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_step, ms_bin = float(ms_t[0]), float(ms_t[1])

    # ---- end to end through the public API with HOST buffers (H2D + D2H inside the timed region)
    e2e = None
    if not args.no_e2e:
        host = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in arrs]
        for hcol, c in zip(host, list(w.axes) + list(w.attrs)):
            hcol.copy_(cols[c].cpu())
        harrs = [db.wrap_tensor(x, mode=db.BIN_ASYNC) for x in host]
        B = int(res.nbins)
        n_out_arrays = 1 + sum(1 for o in w.ops) * len(w.attrs)
        out_host = torch.empty(B * n_out_arrays, dtype=torch.float64).pin_memory()
        he = h
        def e2e_step():
            tt = db.bin_execute(he, harrs[:D], harrs[D:])
            r = db.bin_result(he, tt)  # waits
            ptrs = [r.count] + [getattr(r, k)[a] for a in range(len(w.attrs)) for k in ("sum", "min", "max", "avg")
                                if getattr(r, k)[a]]
            for j, p in enumerate(ptrs):
                db.bin_copy(out_host.data_ptr() + j * B * 8, p, B * 8)
            return len(ptrs) * B * 8
        for _ in range(2):  # warm both staging slots (executes alternate between two slots)
            e2e_step()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        d2h = 0
        for _ in range(args.e2e_steps):
            d2h = e2e_step()
        dt = (time.perf_counter() - t0) / args.e2e_steps
        dt_t = torch.tensor([dt], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(dt_t, op=dist.ReduceOp.MAX)
        dt = float(dt_t[0])
        e2e = {"value": N_total / dt, "unit": UNIT, "h2d_bytes_per_step": n * 8 * len(arrs) * world,
               "d2h_bytes_per_step": d2h * world,
               "host_numa_node": numa_node,
               "note": "public C-ABI bin_execute on pinned host arrays (library stages H2D), results read back D2H"}
        for a in harrs:
            db.bin_array_release(a)

    if rank == 0:
        peak, peak_src = load_peaks()
        bytes_per_row = 8 * (len(w.axes) + len(w.attrs))
        alg_bytes_launch = bytes_per_row * n           # the bin kernel reads every axis/attr column once
        achieved = alg_bytes_launch / (ms_bin * 1e-3) / 1e9 if ms_bin > 0 else 0.0
        B = int(res.nbins)
        out_bytes = B * 8 * (1 + 4 * len(w.attrs))
        step_alg_bytes = bytes_per_row * N_total + out_bytes
        value = N_total / (ms_step * 1e-3)
        if args.evolve:  # the step also ran the producer's KDK kernel: count the library's own phases only
            lib_ms = sum(getattr(prof, "ms_" + k) for k in ("stage", "init", "bounds", "window", "bin", "combine",
                                                            "finalize")) / max(1, prof.executes)
            value = N_total / (lib_ms * 1e-3)
        var = int(prof.variant)
        D = len(w.axes)
        if var & 15 == 4:
            kname = "partition route (k_part_keys, k_part_scan1/2, k_part_scatter[, k_part_refine], k_part_reduce)"
        elif var & 15 == 3:
            kname = "deterministic (k_det_keys, radix passes, k_det_segments, k_det_fold[_long])"
        elif var & 16:
            kname = f"k_bin_fast<{D},1,1,1>" if len(w.attrs) == 1 else f"k_bin_fast<{D},{len(w.attrs)},..>"
        else:
            kname = f"k_bin<{D},..>"
        if world == 1:
            combine = "none (1 rank)"
        elif var & 64:
            combine = "NVLS in-switch combine + finalize (k_combine_nvls: multimem.ld_reduce / multimem.st)"
        elif var & 32:
            combine = "fused NVLink peer-memory combine + finalize (k_combine_peer)"
        else:
            combine = "NCCL allreduce of bin arrays + k_finalize"
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "rows": N_total, "rows_per_rank": n, "res": list(w.res),
                       "bounds": "auto" if args.bounds_auto else [list(w.lo), list(w.hi)],
                       "axes": list(w.axes), "attrs": list(w.attrs), "ops": list(w.ops),
                       "exec": "lockstep (BIN_EXEC_SYNC, stream-ordered)", "deterministic": args.deterministic,
                       "sum_mode": "exact (BIN_SUM_EXACT)" if args.exact else "fast",
                       "l2": "inputs 24 B/row x rows >> 126 MB L2; no flush needed",
                       "inputs": ("evolving: a KDK drift of every row (synth.kdk_step, dt 1e-3) before every execute; "
                                  "value from the library's per-execute phase times") if args.evolve else "fixed",
                       "parallelism": f"dp{world} (contiguous row shards per rank)", "combine": combine},
            "hbm": {"alg_bytes_per_step": step_alg_bytes,
                    "achieved_gbs_step": step_alg_bytes / (ms_step * 1e-3) / 1e9 / world,
                    "frac_of_8TBps_step": step_alg_bytes / (ms_step * 1e-3) / 1e9 / world / NOMINAL_HBM_GBS},
            "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved,
                         "peak": peak, "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak if achieved else None,
                         "traffic": load_traffic(w.name), "ms_per_launch": ms_bin,
                         "alg_bytes_per_launch": alg_bytes_launch,
                         "share_of_step": ms_bin / ms_step if ms_step else None},
            "phases_ms_per_step": {k: getattr(prof, "ms_" + k) / max(1, prof.executes)
                                   for k in ("stage", "init", "bounds", "window", "bin", "combine", "finalize")},
            "gpu_launches": int(prof.kernel_launches),
            "variant": int(prof.variant), "window": list(prof.window)[:len(w.res)],
            "n_in": n_in, "n_out": n_out,
            "clocks": clk.summary(),
        }
        if e2e:
            line["e2e"] = e2e
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(w, args.cpu_seconds)
        print(json.dumps(line), flush=True)

    for a in arrs:
        db.bin_array_release(a)
    db.bin_finalize(h)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
