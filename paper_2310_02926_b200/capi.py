"""ctypes declarations of include/databin.h (argument marshalling only).

Every function here is a direct call into libdatabin.so with the same name
as the C entry point; errors become ``BinError`` carrying the C code and
``bin_last_error()``.  No computation happens in Python.
"""
from __future__ import annotations

import ctypes
import os
import threading

from . import build as _build

# ---- constants (mirror include/databin.h) ----
BIN_OK, BIN_EINVAL, BIN_ESHAPE, BIN_EDTYPE, BIN_EDEVICE, BIN_EDEGENERATE = 0, 1, 2, 3, 4, 5
BIN_ENOMEM, BIN_ENOTSUP, BIN_ECUDA, BIN_ENCCL, BIN_ESTATE = 6, 7, 8, 9, 10
ERROR_NAMES = {0: "BIN_OK", 1: "BIN_EINVAL", 2: "BIN_ESHAPE", 3: "BIN_EDTYPE", 4: "BIN_EDEVICE",
               5: "BIN_EDEGENERATE", 6: "BIN_ENOMEM", 7: "BIN_ENOTSUP", 8: "BIN_ECUDA", 9: "BIN_ENCCL",
               10: "BIN_ESTATE"}
BIN_F64 = 0
BIN_ALLOC_HOST, BIN_ALLOC_HOST_PINNED, BIN_ALLOC_CUDA, BIN_ALLOC_CUDA_ASYNC, BIN_ALLOC_CUDA_UVA, \
    BIN_ALLOC_EXTERNAL = range(6)
BIN_SYNC, BIN_ASYNC = 0, 1
BIN_OP_SUM, BIN_OP_MIN, BIN_OP_MAX, BIN_OP_AVG = 1, 2, 4, 8
OPS = {"sum": BIN_OP_SUM, "min": BIN_OP_MIN, "max": BIN_OP_MAX, "avg": BIN_OP_AVG}
BIN_MAX_DIM, BIN_MAX_ATTR = 3, 16
BIN_EXEC_SYNC, BIN_EXEC_ASYNC, BIN_EXEC_PEER = 0, 1, 2
BIN_DEVICE_HOST, BIN_DEVICE_AUTO = -1, -2
BIN_ROUTE_AUTO, BIN_ROUTE_WINDOW, BIN_ROUTE_PARTITION = 0, 1, 2
ROUTES = {"auto": BIN_ROUTE_AUTO, "window": BIN_ROUTE_WINDOW, "partition": BIN_ROUTE_PARTITION}
BIN_SUM_FAST, BIN_SUM_EXACT = 0, 1


class BinError(RuntimeError):
    def __init__(self, code, fn, msg):
        super().__init__(f"{fn}: {ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code


# ---- structs ----
class bin_spec_t(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int32), ("res", ctypes.c_int32 * 3), ("bounds_auto", ctypes.c_int32),
                ("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3), ("nattr", ctypes.c_int32),
                ("ops", ctypes.c_uint32 * 16), ("deterministic", ctypes.c_int32), ("route", ctypes.c_int32),
                ("sum_mode", ctypes.c_int32)]


class bin_placement_t(ctypes.Structure):
    _fields_ = [("device_id", ctypes.c_int32), ("device_start", ctypes.c_int32),
                ("device_stride", ctypes.c_int32), ("devices_to_use", ctypes.c_int32),
                ("exec", ctypes.c_int32), ("async_snapshot", ctypes.c_int32)]


class bin_comm_t(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("nccl_unique_id", ctypes.c_void_p)]


class bin_result_t(ctypes.Structure):
    _fields_ = [("count", ctypes.c_void_p), ("sum", ctypes.c_void_p * 16), ("min", ctypes.c_void_p * 16),
                ("max", ctypes.c_void_p * 16), ("avg", ctypes.c_void_p * 16), ("nbins", ctypes.c_uint64),
                ("n_in", ctypes.c_uint64), ("n_out", ctypes.c_uint64), ("device", ctypes.c_int32),
                ("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3)]


class bin_profile_t(ctypes.Structure):
    _fields_ = [("ms_bounds", ctypes.c_double), ("ms_init", ctypes.c_double), ("ms_window", ctypes.c_double),
                ("ms_bin", ctypes.c_double), ("ms_combine", ctypes.c_double), ("ms_finalize", ctypes.c_double),
                ("ms_stage", ctypes.c_double), ("executes", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("bin_launches", ctypes.c_int64), ("variant", ctypes.c_int32), ("window", ctypes.c_int32 * 3)]


BIN_MULTI_MAX_OPS, BIN_MULTI_MAX_COLS = 32, 16


class bin_multi_op_t(ctypes.Structure):
    _fields_ = [("spec", bin_spec_t), ("axis_col", ctypes.c_int32 * 3), ("attr_col", ctypes.c_int32 * 16)]


RELEASE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)

_P = ctypes.POINTER
_vp = ctypes.c_void_p
_SIGS = {
    "bin_array_wrap": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int, _vp,
                                      ctypes.c_int, RELEASE_FN, _vp, _P(_vp)]),
    "bin_array_alloc": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int, _vp,
                                       ctypes.c_int, _P(ctypes.c_double), _P(_vp)]),
    "bin_array_data": (ctypes.c_int, [_vp, _P(_vp)]),
    "bin_array_info": (ctypes.c_int, [_vp, _P(ctypes.c_int64), _P(ctypes.c_int32), _P(ctypes.c_int32), _P(_vp)]),
    "bin_array_get_accessible": (ctypes.c_int, [_vp, ctypes.c_int32, _vp, _P(_vp), _P(_vp)]),
    "bin_array_synchronize": (ctypes.c_int, [_vp]),
    "bin_array_release": (None, [_vp]),
    "bin_alloc_stats": (None, [_P(ctypes.c_int64), _P(ctypes.c_int64), _P(ctypes.c_int64)]),
    "bin_placement_default": (None, [_P(bin_placement_t)]),
    "bin_resolve_device": (ctypes.c_int, [_P(bin_placement_t), ctypes.c_int32, ctypes.c_int32, _P(ctypes.c_int32)]),
    "bin_init": (ctypes.c_int, [_P(bin_spec_t), _P(bin_placement_t), _P(bin_comm_t), _P(_vp)]),
    "bin_execute": (ctypes.c_int, [_vp, _P(_vp), ctypes.c_int32, _P(_vp), ctypes.c_int32, _P(ctypes.c_uint64)]),
    "bin_execute_shards": (ctypes.c_int, [_vp, _P(_vp), ctypes.c_int32, _P(_vp), ctypes.c_int32, ctypes.c_int32,
                                          _P(ctypes.c_uint64)]),
    "bin_init_group": (ctypes.c_int, [_P(bin_spec_t), _P(bin_placement_t), ctypes.c_int32, _P(_vp)]),
    "bin_execute_group": (ctypes.c_int, [_P(_vp), ctypes.c_int32, _P(_vp), ctypes.c_int32, _P(_vp), ctypes.c_int32,
                                         _P(ctypes.c_uint64)]),
    "bin_inputs_released": (ctypes.c_int, [_vp, ctypes.c_uint64, _P(_vp)]),
    "bin_wait": (ctypes.c_int, [_vp, ctypes.c_uint64]),
    "bin_result": (ctypes.c_int, [_vp, ctypes.c_uint64, _P(bin_result_t)]),
    "bin_stream": (ctypes.c_int, [_vp, _P(_vp)]),
    "bin_profile_enable": (ctypes.c_int, [_vp, ctypes.c_int32]),
    "bin_profile_read": (ctypes.c_int, [_vp, _P(bin_profile_t)]),
    "bin_finalize": (ctypes.c_int, [_vp]),
    "bin_nccl_unique_id": (ctypes.c_int, [_vp]),
    "bin_copy": (ctypes.c_int, [_vp, _vp, ctypes.c_uint64, _vp]),
    "bin_multi_init": (ctypes.c_int, [_P(bin_multi_op_t), ctypes.c_int32, ctypes.c_int32, _P(bin_placement_t),
                                      _P(bin_comm_t), _P(_vp)]),
    "bin_multi_execute": (ctypes.c_int, [_vp, _P(_vp), ctypes.c_int32, _P(ctypes.c_uint64)]),
    "bin_multi_wait": (ctypes.c_int, [_vp, ctypes.c_uint64]),
    "bin_multi_inputs_released": (ctypes.c_int, [_vp, ctypes.c_uint64, _P(_vp)]),
    "bin_multi_result": (ctypes.c_int, [_vp, ctypes.c_uint64, ctypes.c_int32, _P(bin_result_t)]),
    "bin_multi_profile_enable": (ctypes.c_int, [_vp, ctypes.c_int32]),
    "bin_multi_profile_read": (ctypes.c_int, [_vp, _P(bin_profile_t)]),
    "bin_multi_stream": (ctypes.c_int, [_vp, _P(_vp)]),
    "bin_multi_finalize": (ctypes.c_int, [_vp]),
    "bin_last_error": (ctypes.c_char_p, []),
    "bin_version": (ctypes.c_char_p, []),
}
EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def lib():
    """Loads libdatabin.so from this package directory (building it if stale).

    There is no fallback: if the shared library cannot be built or loaded,
    this raises."""
    global _lib
    with _lock:
        if _lib is None:
            path = _build.LIB
            if os.environ.get("DATABIN_LIB"):          # explicit build variant (A/B experiments)
                path = os.environ["DATABIN_LIB"]
            elif os.environ.get("DATABIN_NO_BUILD") != "1":
                path = _build.build()
            if not os.path.exists(path):
                raise ImportError(f"libdatabin.so missing at {path}; run __graft_entry__.build()")
            L = ctypes.CDLL(path)
            for name, (res, args) in _SIGS.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def check(rc, fn):
    if rc != BIN_OK:
        raise BinError(rc, fn, lib().bin_last_error().decode(errors="replace"))
    return rc
