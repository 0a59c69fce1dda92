"""ctypes front-end of the C oracle (pancake_oracle.c).

TEST INFRASTRUCTURE ONLY -- the parity checker, never the product path.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
``--impl reference`` legs import this module.  Each wrapper names the
reference function it restates (file:line in /root/reference/pkg/src/agentmem).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libpancake_oracle.so")
_lib = None

METRIC_CODES = {"sq_l2": 0, "ip": 1, "cosine": 2}

_f32p = ctypes.POINTER(ctypes.c_float)
_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_i64 = ctypes.c_int64


def build() -> str:
    """Compile the oracle in place (make); returns the library path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        for name in ("or_sq_l2", "or_neg_ip", "or_cosine"):
            getattr(L, name).argtypes = [_f32p, _f32p, _i64, _i64, _f32p]
            getattr(L, name).restype = None
        L.or_distances.argtypes = [_f32p, _f32p, _i64, _i64, ctypes.c_int, _f32p]
        L.or_kmeans_assign.argtypes = [_f32p, _i64, _f32p, _i64, _i64, _i64p, _f64p]
        L.or_centroid.argtypes = [_f32p, _i64, _i64, _f32p]
        L.or_assign_nearest.argtypes = [_f32p, _f32p, _i64p, _i64, _i64, ctypes.c_int]
        L.or_assign_nearest.restype = ctypes.c_int64
        L.or_ivf_search.argtypes = [
            _f32p, _i64p, _i64p, _i64p, _f32p, _i64p, _u8p, _i64, _i64, ctypes.c_int,
            _f32p, _i64, ctypes.c_int, ctypes.c_int, _i64p, _f32p, _i32p, _i64p, _i64p,
            ctypes.c_int,
        ]
        L.or_ivf_search.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def distances(q, mat, metric: str = "sq_l2") -> np.ndarray:
    """core.py:98-109 batch_distances -> kernels.py:73-113 (numba arithmetic)."""
    q, mat = _f32(q), _f32(mat)
    n, d = mat.shape
    out = np.empty(n, dtype=np.float32)
    if n:
        lib().or_distances(_p(q, _f32p), _p(mat, _f32p), n, d, METRIC_CODES[metric], _p(out, _f32p))
    return out


def sq_l2(q, mat):
    """kernels.py:73-83."""
    return distances(q, mat, "sq_l2")


def neg_ip(q, mat):
    """kernels.py:86-95."""
    return distances(q, mat, "ip")


def cosine(q, mat):
    """kernels.py:98-113."""
    return distances(q, mat, "cosine")


def kmeans_assign(x, cents):
    """kernels.py:116-135: labels i64, fp64 distances; ties -> first centroid."""
    x, cents = _f32(x), _f32(cents)
    n, d = x.shape
    labels = np.empty(n, dtype=np.int64)
    dists = np.empty(n, dtype=np.float64)
    lib().or_kmeans_assign(_p(x, _f32p), n, _p(cents, _f32p), len(cents), d, _p(labels, _i64p), _p(dists, _f64p))
    return labels, dists


def centroid(mat) -> np.ndarray:
    """core.py:112-117: fp64 row-order mean cast to fp32."""
    mat = _f32(mat)
    n, d = mat.shape
    out = np.empty(d, dtype=np.float32)
    lib().or_centroid(_p(mat, _f32p), n, d, _p(out, _f32p))
    return out


def assign_nearest(v, cents, cids, metric: str = "sq_l2") -> int:
    """clusters.py:268-279: argmin over candidates, ties -> lower cid."""
    v, cents = _f32(v), _f32(cents)
    cids = np.ascontiguousarray(cids, dtype=np.int64)
    return int(lib().or_assign_nearest(_p(v, _f32p), _p(cents, _f32p), _p(cids, _i64p), len(cids), cents.shape[1], METRIC_CODES[metric]))


class FlatIVF:
    """Arena-form IVF (rows/ids/offsets per list + centroid table) searched by
    the flat restatement of Store._search_read_phase (engine.py:319-426 with
    graph.py:321-396 at exhaustive ef)."""

    def __init__(self, rows, ids, offsets, lengths, cents, cids, metric: str = "sq_l2"):
        self.rows = _f32(rows)
        self.ids = np.ascontiguousarray(ids, dtype=np.int64)
        self.off = np.ascontiguousarray(offsets, dtype=np.int64)
        self.len = np.ascontiguousarray(lengths, dtype=np.int64)
        self.cent = _f32(cents)
        self.cid = np.ascontiguousarray(cids, dtype=np.int64)
        self.metric = metric
        self.d = self.cent.shape[1]

    @classmethod
    def from_lists(cls, lists, cents, cids, metric="sq_l2"):
        """lists: sequence of (ids i64[n], rows f32[n,d])."""
        lens = np.array([len(i) for i, _ in lists], dtype=np.int64)
        off = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
        d = np.asarray(cents).shape[1]
        rows = np.concatenate([np.asarray(r, dtype=np.float32).reshape(-1, d) for _, r in lists])
        ids = np.concatenate([np.asarray(i, dtype=np.int64) for i, _ in lists])
        return cls(rows, ids, off, lens, cents, cids, metric)

    def search(self, Q, nprobe: int, kk: int, in_scope=None, threads: int = 1):
        Q = _f32(Q).reshape(-1, self.d)
        B = len(Q)
        nl = len(self.cid)
        scope = np.ones(nl, dtype=np.uint8) if in_scope is None else np.ascontiguousarray(in_scope, dtype=np.uint8)
        ids = np.full((B, kk), -1, dtype=np.int64)
        dd = np.full((B, kk), np.inf, dtype=np.float32)
        cnt = np.zeros(B, dtype=np.int32)
        probe = np.full((B, nprobe), -1, dtype=np.int64)
        scanned = np.zeros(B, dtype=np.int64)
        lib().or_ivf_search(
            _p(self.rows, _f32p), _p(self.ids, _i64p), _p(self.off, _i64p), _p(self.len, _i64p),
            _p(self.cent, _f32p), _p(self.cid, _i64p), _p(scope, _u8p), nl, self.d,
            METRIC_CODES[self.metric], _p(Q, _f32p), B, nprobe, kk, _p(ids, _i64p), _p(dd, _f32p),
            _p(cnt, _i32p), _p(probe, _i64p), _p(scanned, _i64p), threads,
        )
        return ids, dd, cnt, probe, scanned
