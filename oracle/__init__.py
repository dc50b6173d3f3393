"""CPU oracle for the in situ DataBin hot path (arXiv 2310.02926, Sec. 4.2).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2310_02926_b200`` never imports it.

The arithmetic lives in ``databin_oracle.c`` (plain C, fp64, compiled with
``-O2 -ffp-contract=off``); this module only builds it with gcc and marshals
numpy arrays through ctypes.  See the C file's header for the passages each
function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "databin_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no CUDA, no shared code with the product)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.POINTER
            d_p, u64_p, i32_p = P(ctypes.c_double), P(ctypes.c_uint64), P(ctypes.c_int32)
            dpp = P(P(ctypes.c_double))
            lib.oracle_databin.argtypes = [
                ctypes.c_int, i32_p, ctypes.c_int, d_p, d_p, ctypes.c_int, ctypes.c_int64,
                dpp, ctypes.c_int, dpp, u64_p, d_p, d_p, d_p, d_p, d_p, u64_p, u64_p]
            lib.oracle_databin.restype = ctypes.c_int
            lib.oracle_bounds.argtypes = [ctypes.c_int, ctypes.c_int64, dpp, d_p, d_p]
            lib.oracle_bounds.restype = ctypes.c_int
            lib.oracle_exact_sum.argtypes = [ctypes.c_int64, d_p]
            lib.oracle_exact_sum.restype = ctypes.c_double
            lib.oracle_exact_sums.argtypes = [ctypes.c_int, i32_p, d_p, d_p, ctypes.c_int64, dpp, ctypes.c_int,
                                              dpp, d_p]
            lib.oracle_exact_sums.restype = ctypes.c_int
            u64p = P(ctypes.c_uint64)
            lib.oracle_grid_init.argtypes = [ctypes.c_int64, ctypes.c_int, u64p, d_p, d_p, d_p, d_p]
            lib.oracle_grid_init.restype = None
            lib.oracle_accumulate.argtypes = [ctypes.c_int, i32_p, d_p, d_p, ctypes.c_int64, dpp, ctypes.c_int, dpp,
                                              u64p, d_p, d_p, d_p, d_p, u64p, u64p]
            lib.oracle_accumulate.restype = None
            lib.oracle_merge_into.argtypes = [ctypes.c_int64, ctypes.c_int, u64p, d_p, d_p, d_p, d_p,
                                              u64p, d_p, d_p, d_p, d_p]
            lib.oracle_merge_into.restype = None
            lib.oracle_finalize.argtypes = [ctypes.c_int64, ctypes.c_int, u64p, d_p, d_p]
            lib.oracle_finalize.restype = None
            lib.oracle_bounds_usable.argtypes = [ctypes.c_int, i32_p, d_p, d_p]
            lib.oracle_bounds_usable.restype = ctypes.c_int
            lib.oracle_eq1_device.argtypes = [ctypes.c_int] * 5
            lib.oracle_eq1_device.restype = ctypes.c_int
            _lib = lib
    return _lib


class Degenerate(ValueError):
    """Auto bounds with no usable mesh (the library's BIN_EDEGENERATE)."""


class InvalidArgument(ValueError):
    """Bad arguments, e.g. unusable manual bounds (the library's BIN_EINVAL)."""


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ptr_array(cols):
    arr = (ctypes.POINTER(ctypes.c_double) * max(1, len(cols)))()
    for i, c in enumerate(cols):
        arr[i] = _dptr(c)
    return arr


def _as_f64(cols, n=None):
    out = [np.ascontiguousarray(c, dtype=np.float64) for c in cols]
    for c in out:
        if c.ndim != 1 or (n is not None and c.shape[0] != n):
            raise ValueError("columns must be 1-D and of equal length")
    return out


def databin(axes, attrs, res, lo=None, hi=None, bounds_auto=False, P=1, exact=False):
    """Bin rows (axes[d][i], attrs[a][i]) onto a res[0] x ... mesh.

    Returns a dict with count (u64[B]), sum/sumabs/min/max/avg (f64[A, B]),
    n_in, n_out, lo, hi.  Bins are linearised x fastest (reading R11).
    ``P`` > 1 runs the partition (multi-rank) mode of PAPER.md:479.
    ``exact``: also ``sum_exact`` / ``avg_exact`` -- each bin's exact sum
    rounded once (R20; ``oracle_exact_sums``) and it over count.
    """
    lib = _load()
    ndim = len(axes)
    if not 1 <= ndim <= 3 or len(res) != ndim:
        raise ValueError("1..3 axes with one resolution each")
    n = int(np.asarray(axes[0]).shape[0])
    axes = _as_f64(axes, n)
    attrs = _as_f64(attrs, n)
    nattr = len(attrs)
    resa = np.ascontiguousarray(res, dtype=np.int32)
    B = int(np.prod(resa.astype(np.int64)))
    loa = np.zeros(3, np.float64)
    hia = np.zeros(3, np.float64)
    if not bounds_auto:
        loa[:ndim] = lo
        hia[:ndim] = hi
    count = np.zeros(B, np.uint64)
    shp = (max(nattr, 1), B)
    s, sa, mn, mx, avg = (np.zeros(shp, np.float64) for _ in range(5))
    n_in = ctypes.c_uint64(0)
    n_out = ctypes.c_uint64(0)
    rc = lib.oracle_databin(
        ndim, resa.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), int(bool(bounds_auto)),
        _dptr(loa), _dptr(hia), int(P), n, _ptr_array(axes), nattr, _ptr_array(attrs),
        count.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), _dptr(s), _dptr(sa),
        _dptr(mn), _dptr(mx), _dptr(avg), ctypes.byref(n_in), ctypes.byref(n_out))
    if rc == -1:
        raise Degenerate("auto bounds: no non-NaN row on an axis, or realised bounds not usable (reading R4)")
    if rc == -3:
        raise InvalidArgument("bad arguments or unusable manual bounds (reading R4)")
    if rc != 0:
        raise MemoryError(f"oracle_databin failed rc={rc}")
    k = slice(0, nattr)
    out = dict(count=count, sum=s[k], sumabs=sa[k], min=mn[k], max=mx[k], avg=avg[k],
               n_in=int(n_in.value), n_out=int(n_out.value),
               lo=loa[:ndim].copy(), hi=hia[:ndim].copy())
    if exact:
        se = np.zeros(shp, np.float64)
        rc = lib.oracle_exact_sums(ndim, resa.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _dptr(loa),
                                   _dptr(hia), n, _ptr_array(axes), nattr, _ptr_array(attrs), _dptr(se))
        if rc != 0:
            raise MemoryError("oracle_exact_sums")
        out["sum_exact"] = se[k]
        with np.errstate(invalid="ignore", divide="ignore"):
            out["avg_exact"] = np.where(count > 0, se[k] / np.maximum(count, 1).astype(np.float64), np.nan)
    return out


def databin_blocks(rows, n, res, lo, hi, nattr, P=1, threads=None, chunk=1 << 24):
    """The partition mode of ``databin`` for inputs too large to
    hold at once: ``rows(start, count) -> (axes, attrs)`` produces the columns
    of rows [start, start + count) (e.g. the seeded generator).  Block r of P
    = [floor(rN/P), floor((r+1)N/P)) is fed to ``oracle_accumulate`` chunk by
    chunk in row order into its own grid (one worker thread per block; the C
    call releases the GIL), then the grids are folded in rank order with
    ``oracle_merge_into`` and finished with ``oracle_finalize`` -- the C
    definition of ``oracle_databin(..., P)`` step for step, so the result is
    bit-identical to ``databin(axes, attrs, res, lo, hi, P=P)``.  P = 1 is the
    sequential row-order loop.  Manual bounds only.  Same keys as ``databin``
    (without ``sum_exact``)."""
    from concurrent.futures import ThreadPoolExecutor
    lib = _load()
    ndim = len(res)
    resa = np.ascontiguousarray(res, dtype=np.int32)
    B = int(np.prod(resa.astype(np.int64)))
    loa = np.zeros(3, np.float64)
    hia = np.zeros(3, np.float64)
    loa[:ndim] = lo
    hia[:ndim] = hi
    rp = resa.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    if not lib.oracle_bounds_usable(ndim, rp, _dptr(loa), _dptr(hia)):
        raise InvalidArgument("unusable manual bounds (reading R4)")
    A = max(nattr, 1)
    u64 = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))  # noqa: E731

    def grid():
        g = dict(count=np.empty(B, np.uint64), sum=np.empty((A, B)), sumabs=np.empty((A, B)),
                 min=np.empty((A, B)), max=np.empty((A, B)), n_in=ctypes.c_uint64(0), n_out=ctypes.c_uint64(0))
        lib.oracle_grid_init(B, nattr, u64(g["count"]), _dptr(g["sum"]), _dptr(g["sumabs"]), _dptr(g["min"]),
                             _dptr(g["max"]))
        return g

    def block(r):
        g = grid()
        b0, b1 = r * n // P, (r + 1) * n // P
        for s0 in range(b0, b1, chunk):
            c = min(chunk, b1 - s0)
            axes, attrs = rows(s0, c)
            axes, attrs = _as_f64(axes, c), _as_f64(attrs, c)
            lib.oracle_accumulate(ndim, rp, _dptr(loa), _dptr(hia), c, _ptr_array(axes), nattr, _ptr_array(attrs),
                                  u64(g["count"]), _dptr(g["sum"]), _dptr(g["sumabs"]), _dptr(g["min"]),
                                  _dptr(g["max"]), ctypes.byref(g["n_in"]), ctypes.byref(g["n_out"]))
        return g

    with ThreadPoolExecutor(max_workers=threads or P) as ex:
        parts = list(ex.map(block, range(P)))
    if P == 1:
        out = parts[0]
    else:
        out = grid()
        for g in parts:  # rank order
            lib.oracle_merge_into(B, nattr, u64(out["count"]), _dptr(out["sum"]), _dptr(out["sumabs"]),
                                  _dptr(out["min"]), _dptr(out["max"]), u64(g["count"]), _dptr(g["sum"]),
                                  _dptr(g["sumabs"]), _dptr(g["min"]), _dptr(g["max"]))
            out["n_in"].value += g["n_in"].value
            out["n_out"].value += g["n_out"].value
    avg = np.empty((A, B))
    lib.oracle_finalize(B, nattr, u64(out["count"]), _dptr(out["sum"]), _dptr(avg))
    k = slice(0, nattr)
    return dict(count=out["count"], sum=out["sum"][k], sumabs=out["sumabs"][k], min=out["min"][k],
                max=out["max"][k], avg=avg[k], n_in=int(out["n_in"].value), n_out=int(out["n_out"].value),
                lo=loa[:ndim].copy(), hi=hia[:ndim].copy())


def exact_sum(values) -> float:
    """The exact sum of finite doubles rounded once to nearest-even (R20)."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    return float(_load().oracle_exact_sum(v.shape[0], _dptr(v)))


def bounds(axes):
    """Exact per-axis (min, max) under IEEE totalOrder, before widening."""
    lib = _load()
    n = int(np.asarray(axes[0]).shape[0])
    axes = _as_f64(axes, n)
    lo = np.zeros(3)
    hi = np.zeros(3)
    rc = lib.oracle_bounds(len(axes), n, _ptr_array(axes), _dptr(lo), _dptr(hi))
    if rc != 0:
        raise ValueError("auto bounds of an empty column")
    return lo[:len(axes)].copy(), hi[:len(axes)].copy()


def eq1_device(r, n_u, s, d0, n_a):
    """Eq. (1), read as ((r mod n_u)*s + d0) mod n_a."""
    return int(_load().oracle_eq1_device(r, n_u, s, d0, n_a))
