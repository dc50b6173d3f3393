"""Seeded synthetic particle inputs shared by tests and bench (input only).

This module holds none of the DataBin method's arithmetic: it generates the
columns (x, y, z, mass, vx, vy, vz) of Newton++-shaped particle sets
(uniform with a massive central body, PAPER.md:274-276/:463/:510, and a
Plummer sphere standing in for the clustered MAGI ICs) from a counter-based
hash of (seed, stream, row).  ``synth.cuh`` is compiled for the host (gcc,
-ffp-contract=off) and the device (nvcc, explicit _rn ops) into
``libsynth.so``; ``fill_numpy`` is an independent numpy twin that tests use
to pin both builds bit for bit.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

from .configs import CONFIGS, Workload  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libsynth.so")
_SRCS = [os.path.join(_HERE, f) for f in ("synth.cu", "synth.cuh")]
_lock = threading.Lock()
_lib = None

UNIFORM, PLUMMER = 0, 1
X, Y, Z, M, VX, VY, VZ = range(7)
COLUMNS = {"x": X, "y": Y, "z": Z, "mass": M, "vx": VX, "vy": VY, "vz": VZ}

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false",
              "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-shared", "-std=c++17"]


def build(force: bool = False) -> str:
    newest = max(os.path.getmtime(s) for s in _SRCS)
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", *NVCC_FLAGS, "-o", tmp, _SRCS[0]])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.synth_fill_host.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                                            ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int]
            lib.synth_fill_device.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                                              ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
            lib.synth_kdk_step.argtypes = [ctypes.c_void_p] * 6 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                                                   ctypes.c_double, ctypes.c_double, ctypes.c_void_p]
            lib.synth_direct_step.argtypes = [ctypes.c_void_p] * 7 + [ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                                                      ctypes.c_void_p]
            _lib = lib
    return _lib


def fill_host(dist, central, seed, column, start, n, nthreads=0) -> np.ndarray:
    out = np.empty(int(n), np.float64)
    _load().synth_fill_host(dist, int(central), seed, column, start, int(n), out.ctypes.data, nthreads)
    return out


def fill_device(dist, central, seed, column, start, n, dptr, stream=0) -> None:
    rc = _load().synth_fill_device(dist, int(central), seed, column, start, int(n),
                                   ctypes.c_void_p(dptr), ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"synth_fill_device: cudaError {rc}")


def kdk_step(cols, n, stream=0, central_mass=1000.0, eps2=1e-4, dt=1e-5, start=0):
    """One leapfrog step of the placement-study producer on device columns
    (x, y, z, vx, vy, vz as device pointers) holding global rows start..start+n-1;
    see synth.cu syn_kdk_kernel."""
    rc = _load().synth_kdk_step(*[ctypes.c_void_p(c) for c in cols], int(n), int(start), central_mass, eps2, dt,
                                ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"synth_kdk_step: cudaError {rc}")


def direct_step(cols, n, stream=0, eps2=1e-4, dt=1e-6):
    """One O(N^2) direct-sum gravity step (the Newton++ solver class) on device
    columns (x, y, z, vx, vy, vz, mass as device pointers); synth.cu."""
    rc = _load().synth_direct_step(*[ctypes.c_void_p(c) for c in cols], int(n), eps2, dt, ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"synth_direct_step: cudaError {rc}")


# ---------------------------------------------------------------- numpy twin
_M1, _M2 = np.uint64(0xbf58476d1ce4e5b9), np.uint64(0x94d049bb133111eb)
_G, _K2, _K3 = np.uint64(0x9E3779B97F4A7C15), np.uint64(0xD1B54A32D192ED03), np.uint64(0x632BE59BD9B4E019)


def _mix64(z):
    z = z ^ (z >> np.uint64(30))
    z = z * _M1
    z = z ^ (z >> np.uint64(27))
    z = z * _M2
    return z ^ (z >> np.uint64(31))


def _u01(seed, stream, idx):
    with np.errstate(over="ignore"):
        k = _mix64(np.uint64(seed) * _G + np.uint64(stream) * _K2 + _K3)
        z = _mix64(k + (idx + np.uint64(1)) * _G)
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def _uniform(seed, stream, idx, a, b):
    return a + (b - a) * _u01(seed, stream, idx)


def fill_numpy(dist, central, seed, column, start, n) -> np.ndarray:
    """Independent numpy implementation of synth.cuh (same bits)."""
    idx = np.arange(start, start + n, dtype=np.uint64)
    if column == M:
        out = _uniform(seed, 200, idx, 0.5, 1.5)
    elif column in (VX, VY, VZ):
        out = _uniform(seed, 210 + column - VX, idx, -1.0, 1.0)
    elif dist == UNIFORM:
        out = _uniform(seed, 220 + column, idx, -1.0, 1.0)
    else:
        t = np.maximum(np.maximum(_u01(seed, 0, idx), _u01(seed, 1, idx)), _u01(seed, 2, idx))
        t = 0.9996 * t
        r = t / np.sqrt(1.0 - t * t)
        a = np.ones(n)
        b = np.zeros(n)
        c = np.zeros(n)
        s = np.ones(n)
        todo = np.arange(n)
        for k in range(32):
            if todo.size == 0:
                break
            ii = idx[todo]
            aa = _uniform(seed, 8 + 3 * k, ii, -1.0, 1.0)
            bb = _uniform(seed, 8 + 3 * k + 1, ii, -1.0, 1.0)
            cc = _uniform(seed, 8 + 3 * k + 2, ii, -1.0, 1.0)
            ss = (aa * aa + bb * bb) + cc * cc
            ok = (ss > 1e-12) & (ss <= 1.0)
            sel = todo[ok]
            a[sel], b[sel], c[sel], s[sel] = aa[ok], bb[ok], cc[ok], ss[ok]
            todo = todo[~ok]
        f = r / np.sqrt(s)
        out = (a, b, c)[column] * f
    if dist == UNIFORM and central and start == 0 and n > 0:
        out[0] = 1000.0 if column == M else 0.0
    return out
