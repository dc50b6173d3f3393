"""Host NUMA placement for pinned staging buffers (host plumbing, no method arithmetic).

The host-placement path of the paper's array handle (HAMR) stages
pinned host columns into device memory; on a multi-socket box a pinned page on
the socket far from the GPU's PCIe root crosses the socket link on every H2D
copy.  `bind_to_gpu(i)` moves the calling thread (and the threads it creates
afterwards) onto the CPUs of GPU i's NUMA node and prefers that node for new
pages, so pinned buffers touched afterwards are local to the GPU.  Call it
before the first pinned allocation (bench.py does it before importing torch).
Every function is a no-op on single-node hosts or when sysfs/NVML are absent.
"""
from __future__ import annotations

import ctypes
import glob
import os
import platform

_SYS_SET_MEMPOLICY = {"x86_64": 238, "aarch64": 237}
_MPOL_PREFERRED = 1


def _parse_cpulist(s: str) -> list[int]:
    out: list[int] = []
    for part in s.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            out.extend(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


def node_cpus(node: int) -> list[int]:
    try:
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            return _parse_cpulist(f.read())
    except OSError:
        return []


def cpu_nodes() -> list[int]:
    """NUMA nodes that have CPUs."""
    nodes = []
    for p in sorted(glob.glob("/sys/devices/system/node/node[0-9]*")):
        n = int(os.path.basename(p)[4:])
        if node_cpus(n):
            nodes.append(n)
    return nodes


def _nvml_handle(index: int):
    import pynvml
    pynvml.nvmlInit()
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ent = [v.strip() for v in vis.split(",") if v.strip()]
        if index < len(ent):
            e = ent[index]
            if e.isdigit():
                return pynvml.nvmlDeviceGetHandleByIndex(int(e))
            return pynvml.nvmlDeviceGetHandleByUUID(e)
    return pynvml.nvmlDeviceGetHandleByIndex(index)


def node_of_gpu(index: int) -> int:
    """NUMA node of CUDA device `index`'s PCIe function, -1 if unknown."""
    try:
        import pynvml
        bus = pynvml.nvmlDeviceGetPciInfo(_nvml_handle(index)).busId
        bus = bus.decode() if isinstance(bus, bytes) else bus
        dom, rest = bus.split(":", 1)
        path = f"/sys/bus/pci/devices/{int(dom, 16):04x}:{rest.lower()}/numa_node"
        with open(path) as f:
            return int(f.read().strip())
    except Exception:  # noqa: BLE001
        return -1


def bind_to_node(node: int) -> bool:
    """Pin the calling thread to `node`'s CPUs and prefer `node` for new pages."""
    cpus = node_cpus(node)
    if not cpus:
        return False
    allowed = os.sched_getaffinity(0)
    use = [c for c in cpus if c in allowed] or cpus
    try:
        os.sched_setaffinity(0, use)
    except OSError:
        return False
    nr = _SYS_SET_MEMPOLICY.get(platform.machine())
    if nr is not None and node < 64:
        try:
            libc = ctypes.CDLL(None, use_errno=True)
            mask = ctypes.c_ulong(1 << node)
            libc.syscall(nr, _MPOL_PREFERRED, ctypes.byref(mask), ctypes.c_ulong(64))
        except Exception:  # noqa: BLE001
            pass
    return True


def bind_to_gpu(index: int) -> int:
    """bind_to_node(node_of_gpu(index)) when the host has more than one NUMA node; returns the node or -1."""
    if len(cpu_nodes()) < 2:
        return -1
    node = node_of_gpu(index)
    if node < 0:
        return -1
    return node if bind_to_node(node) else -1
