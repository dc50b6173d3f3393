"""Pinned host -> device copy bandwidth as a function of where the pinned pages
and the copying thread live (NUMA node).  Explains the spread of bench.py's
`e2e` number (PCIe-bound: 2.4 GB of inputs per C3 step) across boxes.

Usage: python tools/h2d_numa_probe.py [--gpu 0] [--mb 800]
Prints one JSON line per NUMA node with CPUs, plus the unbound case.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def child(node, gpu, mb):
    from paper_2310_02926_b200.numa import bind_to_node, node_of_gpu  # noqa: F401
    if node >= 0:
        bind_to_node(node)
    import torch
    dev = torch.device("cuda", gpu)
    n = mb * (1 << 20) // 8
    h = torch.empty(n, dtype=torch.float64).pin_memory()
    h.fill_(1.0)  # first touch on this thread's node
    d = torch.empty(n, dtype=torch.float64, device=dev)
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        for _ in range(2):
            d.copy_(h, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(5):
            d.copy_(h, non_blocking=True)
        e1.record(s)
    e1.synchronize()
    gbs = 5 * n * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9
    print(json.dumps({"node": node, "gpu": gpu, "gpu_node": node_of_gpu(gpu), "mb": mb, "h2d_gbs": round(gbs, 2),
                      "cpus": len(os.sched_getaffinity(0))}), flush=True)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpu", type=int, default=0)
    p.add_argument("--mb", type=int, default=800)
    p.add_argument("--child", type=int, default=None)
    a = p.parse_args()
    if a.child is not None:
        child(a.child, a.gpu, a.mb)
        return
    from paper_2310_02926_b200.numa import cpu_nodes
    for node in [-1] + cpu_nodes():
        subprocess.run([sys.executable, __file__, "--gpu", str(a.gpu), "--mb", str(a.mb), "--child", str(node)],
                       check=False)


if __name__ == "__main__":
    main()
