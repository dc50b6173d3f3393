#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py full  gpurun_out/prof_kbin_X.ncu-rep  > profiles/rNN_kbin_X.txt
    python tools/ncu_summary.py launches gpurun_out/launches_X.csv     > profiles/rNN_launches_X.txt
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum",
        "smsp__inst_executed_op_shared_atom.sum", "smsp__inst_executed_op_global_red.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "sm__cycles_elapsed.avg.per_second"]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = OrderedDict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"kernel: {d.get('Kernel Name')}  grid={d.get('launch__grid_size')} block={d.get('launch__block_size')}")
        for k in KEYS:
            if k in d:
                print(f"  {k:78s} {d[k]:>18s} {u.get(k, '')}")
    det = subprocess.run(["ncu", "-i", path, "--page", "details"], capture_output=True, text=True).stdout
    keep = [ln for ln in det.splitlines() if any(s in ln for s in (
        "Duration", "Throughput", "Busy", "Eligible", "Active Threads", "Issued Ipc", "Warp Cycles Per Issued",
        "Hit Rate", "Registers", "Shared Memory Per Block", "Achieved Occupancy"))]
    print("\n-- details (selected lines) --")
    print("\n".join(keep))


def launches(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = OrderedDict()
    for r in rows[1:]:
        name = r[ki]
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for k, v in agg.items() if "syn_fill" not in k)
    print("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)")
    print(f"{'kernel':70s} {'n':>4s} {'avg_us':>10s} {'share_of_step':>14s}")
    for k, v in agg.items():
        share = "" if "syn_fill" in k else f"{sum(v) / tot:14.3f}"
        print(f"{k[:70]:70s} {len(v):4d} {sum(v) / len(v) / 1e3:10.1f} {share}")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
