"""ctypes binding of libpancake_b200.so (the C-ABI in include/pancake_b200.h).

There is no fallback: if the shared library is missing or no CUDA device is
present, every entry point raises.  Build it with ``__graft_entry__.build()``
(or ``python -m paper_2602_21477_b200.build``).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .core import AcceleratorError, UsageError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpancake_b200.so")

PK_OK = 0
PK_ERR_USAGE = 1
PK_ERR_DEVICE = 2
PK_ERR_NOMEM = 3
PK_DEVICE_PTRS = 1
PK_ASYNC_SLOTS = 4  # include/pancake_b200.h
KKMAX = 64
NPROBE_MAX = 2048

_f32p = ctypes.POINTER(ctypes.c_float)
_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_int = ctypes.c_int
_vp = ctypes.c_void_p

# (name, argtypes, restype)
_SIGS = [
    ("pk_last_error", [], ctypes.c_char_p),
    ("pk_version", [], _int),
    ("pk_device_count", [_i32p], _int),
    ("pk_distances", [_vp, _i64, _vp, _i64, _i64, _int, _vp, _int], _int),
    ("pk_kmeans_assign", [_vp, _i64, _vp, _i64, _i64, _vp, _vp, _int], _int),
    ("pk_centroid", [_vp, _i64, _i64, _vp, _int], _int),
    ("pk_centroids_segmented", [_vp, _i64, _i64, _vp, _i64, _vp, _int], _int),
    ("pk_index_create", [_i64, _int, _int, _i64, _i64, ctypes.POINTER(_vp)], _int),
    ("pk_index_destroy", [_vp], _int),
    ("pk_sync", [_vp], _int),
    ("pk_stream", [_vp], _vp),
    ("pk_index_bytes", [_vp, _i64p], _int),
    ("pk_list_create", [_vp, _i64, _i32, _vp, _vp, _i64, _vp, _int], _int),
    ("pk_list_append", [_vp, _i64, _vp, _vp, _i64, _int], _int),
    ("pk_list_append_batch", [_vp, _i64, _vp, _vp, _vp], _int),
    ("pk_list_remove_row", [_vp, _i64, _i64], _int),
    ("pk_list_retire", [_vp, _i64], _int),
    ("pk_list_recompute", [_vp, _i64, _vp], _int),
    ("pk_list_set_centroid", [_vp, _i64, _vp], _int),
    ("pk_list_size", [_vp, _i64, _i64p], _int),
    ("pk_list_read", [_vp, _i64, _vp, _vp], _int),
    ("pk_search", [_vp, _vp, _i64, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _int], _int),
    ("pk_assign", [_vp, _vp, _i64, _i32, _vp, _vp, _int], _int),
    ("pk_profile_begin", [_vp], _int),
    ("pk_profile_end", [_vp, _vp, _int, _i32p], _int),
    ("pk_debug_pool_counts", [_vp, _vp, _i64], _int),
    ("pk_debug_coarse_counts", [_vp, _vp, _i64], _int),
    ("pk_debug_fail_next_alloc", [_vp, _int], _int),
    ("pk_debug_rerank_counts", [_vp, _vp, _i64], _int),
    ("pk_search_coarse", [_vp, _vp, _i64, _vp, _i32, _i32, _vp, _int], _int),
    ("pk_search_probed", [_vp, _vp, _i64, _vp, _i32, _i32, _i64, _vp, _int], _int),
    ("pk_index_enable_tier", [_vp, _i64], _int),
    ("pk_list_set_resident", [_vp, _i64, _int], _int),
    ("pk_list_residency", [_vp, _i64, ctypes.POINTER(_int)], _int),
    ("pk_tier_stats", [_vp, _vp, _int], _int),
    ("pk_search_coarse_cids", [_vp, _vp, _i64, _vp, _i32, _i32, _vp], _int),
    ("pk_scan_lists", [_vp, _vp, _vp, _i32, _vp, _vp, _vp], _int),
    ("pk_combine_create", [_vp, _i32, _i32, _i64, _i32, _vp], _int),
    ("pk_combine_open", [_vp, _i32, _vp, _vp], _int),
    ("pk_combine_area", [_vp], _vp),
    ("pk_combine_search_probed", [_vp, _vp, _i64, _vp, _i32, _i64, _int], _int),
    ("pk_combine_merge", [_vp, _i64, ctypes.c_double, _vp, _vp, _vp, _vp, _vp, _int], _int),
    ("pk_combine_status", [_vp, _vp], _int),
    ("pk_search_submit", [_vp, _i32, _vp, _i64, _vp, _i32, _i32, _i32], _int),
    ("pk_search_collect", [_vp, _i32, _vp, _vp, _vp, _vp, _vp], _int),
    ("pk_list_add_remote", [_vp, _i64, _i32, _vp], _int),
    ("pk_shard_block_bytes", [_i64, _i32], _i64),
    ("pk_merge_shards", [_vp, _vp, _i32, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _int], _int),
    ("pk_graph_set", [_vp, _i32, _i64, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp], _int),
    ("pk_search_graph", [_vp, _vp, _i64, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp,
                         _vp, _vp, _int], _int),
    ("pk_graph_probe", [_vp, _vp, _i64, _vp, _i32, _i32, _i32, _i32, _vp, _vp], _int),
    ("pk_centroid_dists", [_vp, _vp, _i64, _vp, _vp], _int),
    ("pk_list_slot", [_vp, _i64, _i32p], _int),
    ("pk_slot_count", [_vp, _i32p], _int),
    ("pk_rows_put", [_vp, _vp, _vp, _i64], _int),
    ("pk_agent_read", [_vp, _vp, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _i32, _vp, _i32, _vp, _vp, _i32,
                       _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _i64], _int),
    ("pk_l1_place", [_vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp], _int),
    ("pk_agent_lists", [_vp, _vp, _i64, _vp, _i32, _i32, _i32, _i32, _i64, _vp, _vp, _vp, _vp, _vp, _vp], _int),
    ("pk_list_version", [_vp, _vp], _int),
    ("pk_rows_reserve", [_vp, _i64], _int),
]
STAGES = ("input", "coarse_dist", "coarse_select", "route", "scan", "merge_out")
EXPORTED = [s[0] for s in _SIGS]

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load and type the library (no device work)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise AcceleratorError(
                    f"native library not built: {path} is missing "
                    "(run __graft_entry__.build()); there is no CPU fallback"
                )
            lib = ctypes.CDLL(path)
            for name, args, res in _SIGS:
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


def lib():
    return _lib if _lib is not None else load()


def check(rc: int):
    if rc == PK_OK:
        return
    msg = lib().pk_last_error().decode(errors="replace")
    if rc == PK_ERR_USAGE:
        raise UsageError(msg)
    raise AcceleratorError(msg)


def ptr(a) -> int | None:
    """Raw data pointer of a numpy array (C-contiguous) or torch tensor."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch tensor (device pointer with PK_DEVICE_PTRS)


def f32(a, d: int | None = None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    if d is not None:
        a = a.reshape(-1, d)
    return a


def device_count() -> int:
    n = ctypes.c_int32(0)
    check(lib().pk_device_count(ctypes.byref(n)))
    return int(n.value)
