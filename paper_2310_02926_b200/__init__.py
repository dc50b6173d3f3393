"""B200-native in situ DataBin (arXiv 2310.02926, Sec. 4.2) -- Python binding.

The hot path lives in ``libdatabin.so`` (hand-written sm_100a CUDA + NCCL,
``csrc/``) behind the C ABI of ``include/databin.h``.  This package is a thin
ctypes layer with the same names (``bin_array_wrap``, ``bin_init``,
``bin_execute``, ``bin_wait``, ``bin_result``, ``bin_finalize``, ...), plus
helpers that marshal torch tensors (device memory, streams) and numpy arrays
into the C calls.  No binning step runs in Python and there is no CPU
fallback: if the library is missing the import fails.
"""
from __future__ import annotations

import ctypes

import numpy as np

from .capi import (  # noqa: F401
    BIN_ALLOC_CUDA, BIN_ALLOC_CUDA_ASYNC, BIN_ALLOC_CUDA_UVA, BIN_ALLOC_EXTERNAL, BIN_ALLOC_HOST,
    BIN_ALLOC_HOST_PINNED, BIN_ASYNC, BIN_DEVICE_AUTO, BIN_DEVICE_HOST, BIN_EXEC_ASYNC, BIN_EXEC_PEER,
    BIN_EXEC_SYNC, BIN_F64, BIN_OP_AVG, BIN_OP_MAX, BIN_OP_MIN, BIN_OP_SUM, BIN_ROUTE_AUTO, BIN_ROUTE_PARTITION,
    BIN_ROUTE_WINDOW, BIN_SUM_EXACT, BIN_SUM_FAST, BIN_SYNC, EXPORTED, OPS, ROUTES,
    BIN_MULTI_MAX_COLS, BIN_MULTI_MAX_OPS, RELEASE_FN, BinError, bin_comm_t, bin_multi_op_t, bin_placement_t, bin_profile_t, bin_result_t, bin_spec_t, check, lib)

_lib = lib()  # load (and build if stale) at import: no silent fallback


# ---------------------------------------------------------------- array handle
def bin_array_wrap(ptr, n, device, alloc=BIN_ALLOC_EXTERNAL, stream=0, mode=BIN_ASYNC, release=None,
                   release_ctx=None, dtype=BIN_F64):
    """Zero-copy wrap; ``release`` is a RELEASE_FN (keep a reference to it)."""
    out = ctypes.c_void_p()
    cb = release if release is not None else RELEASE_FN()
    check(_lib.bin_array_wrap(ctypes.c_void_p(ptr), int(n), dtype, int(device), int(alloc),
                              ctypes.c_void_p(stream), int(mode), cb, ctypes.c_void_p(release_ctx),
                              ctypes.byref(out)), "bin_array_wrap")
    return out.value


def bin_array_alloc(n, device, alloc, stream=0, mode=BIN_SYNC, fill=None, dtype=BIN_F64):
    out = ctypes.c_void_p()
    f = ctypes.byref(ctypes.c_double(fill)) if fill is not None else None
    check(_lib.bin_array_alloc(int(n), dtype, int(device), int(alloc), ctypes.c_void_p(stream), int(mode), f,
                               ctypes.byref(out)), "bin_array_alloc")
    return out.value


def bin_array_data(a):
    p = ctypes.c_void_p()
    check(_lib.bin_array_data(ctypes.c_void_p(a), ctypes.byref(p)), "bin_array_data")
    return p.value or 0


def bin_array_info(a):
    n, dev, al, st = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_void_p()
    check(_lib.bin_array_info(ctypes.c_void_p(a), ctypes.byref(n), ctypes.byref(dev), ctypes.byref(al),
                              ctypes.byref(st)), "bin_array_info")
    return dict(n=n.value, device=dev.value, alloc=al.value, stream=st.value or 0)


def bin_array_get_accessible(a, device, stream=0):
    p, v = ctypes.c_void_p(), ctypes.c_void_p()
    check(_lib.bin_array_get_accessible(ctypes.c_void_p(a), int(device), ctypes.c_void_p(stream),
                                        ctypes.byref(p), ctypes.byref(v)), "bin_array_get_accessible")
    return p.value or 0, v.value


def bin_array_synchronize(a):
    check(_lib.bin_array_synchronize(ctypes.c_void_p(a)), "bin_array_synchronize")


def bin_array_release(a):
    if a:
        _lib.bin_array_release(ctypes.c_void_p(a))


def bin_alloc_stats():
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.bin_alloc_stats(ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
    return dict(live=a.value, total=b.value, live_bytes=c.value)


# ---------------------------------------------------------------- operator
def make_spec(res, lo=None, hi=None, nattr=0, ops=("sum", "min", "max", "avg"), bounds_auto=False,
              deterministic=False, route="auto", exact=False) -> bin_spec_t:
    """Builds a bin_spec_t; ``ops`` is one op tuple for all attributes or a list per attribute."""
    s = bin_spec_t()
    s.ndim = len(res)
    for d, r in enumerate(res):
        s.res[d] = int(r)
        if not bounds_auto:
            s.lo[d] = float(lo[d])
            s.hi[d] = float(hi[d])
    s.bounds_auto = int(bool(bounds_auto))
    s.nattr = int(nattr)
    per = ops if (nattr and isinstance(ops, (list,)) and len(ops) == nattr and not isinstance(ops[0], str)) \
        else [ops] * nattr
    for a in range(nattr):
        m = 0
        for o in per[a]:
            m |= OPS[o]
        s.ops[a] = m
    s.deterministic = int(bool(deterministic))
    s.route = ROUTES[route] if isinstance(route, str) else int(route)
    s.sum_mode = BIN_SUM_EXACT if exact else BIN_SUM_FAST
    return s


def make_placement(device_id=BIN_DEVICE_AUTO, device_start=0, device_stride=1, devices_to_use=0,
                   exec=BIN_EXEC_SYNC, async_snapshot=1) -> bin_placement_t:
    p = bin_placement_t()
    p.device_id, p.device_start, p.device_stride = device_id, device_start, device_stride
    p.devices_to_use, p.exec, p.async_snapshot = devices_to_use, exec, async_snapshot
    return p


def bin_placement_default() -> bin_placement_t:
    p = bin_placement_t()
    _lib.bin_placement_default(ctypes.byref(p))
    return p


def bin_resolve_device(placement, rank, n_avail):
    d = ctypes.c_int32()
    check(_lib.bin_resolve_device(ctypes.byref(placement), int(rank), int(n_avail), ctypes.byref(d)),
          "bin_resolve_device")
    return d.value


def bin_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(_lib.bin_nccl_unique_id(buf), "bin_nccl_unique_id")
    return buf.raw


def bin_init(spec, placement=None, rank=0, nranks=1, nccl_id: bytes | None = None):
    comm = bin_comm_t()
    comm.rank, comm.nranks = rank, nranks
    idbuf = None
    if nccl_id is not None:
        idbuf = ctypes.create_string_buffer(nccl_id, 128)
        comm.nccl_unique_id = ctypes.cast(idbuf, ctypes.c_void_p)
    out = ctypes.c_void_p()
    pl = ctypes.byref(placement) if placement is not None else None
    check(_lib.bin_init(ctypes.byref(spec), pl, ctypes.byref(comm), ctypes.byref(out)), "bin_init")
    return out.value


def bin_execute(h, axes, attrs):
    ax = (ctypes.c_void_p * max(1, len(axes)))(*axes)
    at = (ctypes.c_void_p * max(1, len(attrs)))(*attrs)
    t = ctypes.c_uint64()
    check(_lib.bin_execute(ctypes.c_void_p(h), ax, len(axes), at, len(attrs), ctypes.byref(t)), "bin_execute")
    return t.value


def bin_execute_shards(h, shards):
    """shards: list of (axes, attrs) handle lists, one per row block (fan-in)."""
    ax = [a for axes, _ in shards for a in axes]
    at = [a for _, attrs in shards for a in attrs]
    naxes, nattr = len(shards[0][0]), len(shards[0][1])
    axa = (ctypes.c_void_p * max(1, len(ax)))(*ax)
    ata = (ctypes.c_void_p * max(1, len(at)))(*at)
    t = ctypes.c_uint64()
    check(_lib.bin_execute_shards(ctypes.c_void_p(h), axa, naxes, ata, nattr, len(shards), ctypes.byref(t)),
          "bin_execute_shards")
    return t.value


def bin_init_group(spec, nranks, placement=None):
    """nranks handles (ranks 0..nranks-1) of a one-device rank group."""
    out = (ctypes.c_void_p * int(nranks))()
    pl = ctypes.byref(placement) if placement is not None else None
    check(_lib.bin_init_group(ctypes.byref(spec), pl, int(nranks), out), "bin_init_group")
    return [x for x in out]


def bin_execute_group(hs, shards):
    """shards[r] = (axes, attrs) array handles of rank r; returns the shared ticket."""
    ax = [a for axes, _ in shards for a in axes]
    at = [a for _, attrs in shards for a in attrs]
    naxes, nattr = len(shards[0][0]), len(shards[0][1])
    ha = (ctypes.c_void_p * len(hs))(*hs)
    axa = (ctypes.c_void_p * max(1, len(ax)))(*ax)
    ata = (ctypes.c_void_p * max(1, len(at)))(*at)
    t = ctypes.c_uint64()
    check(_lib.bin_execute_group(ha, len(hs), axa, naxes, ata, nattr, ctypes.byref(t)), "bin_execute_group")
    return t.value


def bin_inputs_released(h, ticket):
    ev = ctypes.c_void_p()
    check(_lib.bin_inputs_released(ctypes.c_void_p(h), ticket, ctypes.byref(ev)), "bin_inputs_released")
    return ev.value


def bin_wait(h, ticket):
    check(_lib.bin_wait(ctypes.c_void_p(h), ticket), "bin_wait")


def bin_result(h, ticket) -> bin_result_t:
    r = bin_result_t()
    check(_lib.bin_result(ctypes.c_void_p(h), ticket, ctypes.byref(r)), "bin_result")
    return r


def bin_stream(h):
    s = ctypes.c_void_p()
    check(_lib.bin_stream(ctypes.c_void_p(h), ctypes.byref(s)), "bin_stream")
    return s.value or 0


def bin_profile_enable(h, on=True):
    check(_lib.bin_profile_enable(ctypes.c_void_p(h), int(bool(on))), "bin_profile_enable")


def bin_profile_read(h) -> bin_profile_t:
    p = bin_profile_t()
    check(_lib.bin_profile_read(ctypes.c_void_p(h), ctypes.byref(p)), "bin_profile_read")
    return p


def bin_finalize(h):
    check(_lib.bin_finalize(ctypes.c_void_p(h)), "bin_finalize")


def bin_copy(dst, src, nbytes, stream=0):
    check(_lib.bin_copy(ctypes.c_void_p(dst), ctypes.c_void_p(src), int(nbytes), ctypes.c_void_p(stream)),
          "bin_copy")


def bin_last_error() -> str:
    return _lib.bin_last_error().decode(errors="replace")


def bin_version() -> str:
    return _lib.bin_version().decode()


# ---------------------------------------------------------------- fused multi-operator (bin_multi_*)
def make_multi_op(spec: bin_spec_t, axis_col, attr_col=()) -> bin_multi_op_t:
    """One instance of a fused set: its spec plus indices into the shared column list."""
    o = bin_multi_op_t()
    o.spec = spec
    for d, c in enumerate(axis_col):
        o.axis_col[d] = int(c)
    for a, c in enumerate(attr_col):
        o.attr_col[a] = int(c)
    return o


def bin_multi_init(ops, ncols, placement=None, rank=0, nranks=1, nccl_id: bytes | None = None):
    arr = (bin_multi_op_t * len(ops))(*ops)
    comm = bin_comm_t()
    comm.rank, comm.nranks = rank, nranks
    idbuf = None
    if nccl_id is not None:
        idbuf = ctypes.create_string_buffer(nccl_id, 128)
        comm.nccl_unique_id = ctypes.cast(idbuf, ctypes.c_void_p)
    out = ctypes.c_void_p()
    pl = ctypes.byref(placement) if placement is not None else None
    check(_lib.bin_multi_init(arr, len(ops), int(ncols), pl, ctypes.byref(comm), ctypes.byref(out)),
          "bin_multi_init")
    return out.value


def bin_multi_execute(m, cols):
    c = (ctypes.c_void_p * max(1, len(cols)))(*cols)
    t = ctypes.c_uint64()
    check(_lib.bin_multi_execute(ctypes.c_void_p(m), c, len(cols), ctypes.byref(t)), "bin_multi_execute")
    return t.value


def bin_multi_inputs_released(m, ticket):
    ev = ctypes.c_void_p()
    check(_lib.bin_multi_inputs_released(ctypes.c_void_p(m), ticket, ctypes.byref(ev)), "bin_multi_inputs_released")
    return ev.value


def bin_multi_wait(m, ticket):
    check(_lib.bin_multi_wait(ctypes.c_void_p(m), ticket), "bin_multi_wait")


def bin_multi_result(m, ticket, op) -> bin_result_t:
    r = bin_result_t()
    check(_lib.bin_multi_result(ctypes.c_void_p(m), ticket, int(op), ctypes.byref(r)), "bin_multi_result")
    return r


def bin_multi_profile_enable(m, on=True):
    check(_lib.bin_multi_profile_enable(ctypes.c_void_p(m), int(bool(on))), "bin_multi_profile_enable")


def bin_multi_profile_read(m) -> bin_profile_t:
    p = bin_profile_t()
    check(_lib.bin_multi_profile_read(ctypes.c_void_p(m), ctypes.byref(p)), "bin_multi_profile_read")
    return p


def bin_multi_stream(m):
    s = ctypes.c_void_p()
    check(_lib.bin_multi_stream(ctypes.c_void_p(m), ctypes.byref(s)), "bin_multi_stream")
    return s.value or 0


def bin_multi_finalize(m):
    check(_lib.bin_multi_finalize(ctypes.c_void_p(m)), "bin_multi_finalize")


# ---------------------------------------------------------------- marshalling helpers
def wrap_tensor(t, stream=None, mode=BIN_ASYNC):
    """Zero-copy bin_array for a contiguous float64 torch tensor (borrowed)."""
    import torch
    if t.dtype != torch.float64 or not t.is_contiguous() or t.dim() != 1:
        raise BinError(3, "wrap_tensor", "need a contiguous 1-D float64 tensor")
    if t.is_cuda:
        s = stream if stream is not None else torch.cuda.current_stream(t.device).cuda_stream
        return bin_array_wrap(t.data_ptr(), t.numel(), t.device.index, BIN_ALLOC_EXTERNAL, s, mode)
    alloc = BIN_ALLOC_HOST_PINNED if t.is_pinned() else BIN_ALLOC_HOST
    return bin_array_wrap(t.data_ptr(), t.numel(), -1, alloc, stream or 0, mode)


def wrap_numpy(a: np.ndarray, mode=BIN_SYNC):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return bin_array_wrap(a.ctypes.data, a.shape[0], -1, BIN_ALLOC_HOST, 0, mode), a


def result_to_numpy(h, ticket, spec: bin_spec_t, op=None) -> dict:
    """Copies one execute's outputs to host numpy arrays (D2H through bin_copy).
    With ``op`` set, ``h`` is a bin_multi handle and instance ``op`` is read."""
    r = bin_result(h, ticket) if op is None else bin_multi_result(h, ticket, op)
    B = int(r.nbins)
    out = dict(n_in=int(r.n_in), n_out=int(r.n_out), lo=np.array(r.lo[:spec.ndim]),
               hi=np.array(r.hi[:spec.ndim]), device=r.device)
    cnt = np.empty(B, np.uint64)
    bin_copy(cnt.ctypes.data, r.count, B * 8)
    out["count"] = cnt
    for key in ("sum", "min", "max", "avg"):
        arrs = []
        for a in range(spec.nattr):
            p = getattr(r, key)[a]
            if p:
                x = np.empty(B, np.float64)
                bin_copy(x.ctypes.data, p, B * 8)
                arrs.append(x)
            else:
                arrs.append(None)
        out[key] = arrs
    return out
