"""Kernel table, device-backed: the replacement of ``kernels.BACKENDS``
(ref/kernels.py:138-158) and ``core.batch_distances`` / ``centroid`` /
``deviation`` (ref/core.py:89-134).

Same names, argument meaning and results (bit-identical to the reference's
active numba backend), computed by the sm_100a kernels behind the C-ABI.
There is no numpy fallback and no backend switch.
"""

from __future__ import annotations

import numpy as np

from . import _native as N


def _metric_code(metric) -> int:
    from .core import Metric

    if isinstance(metric, Metric):
        return metric.wire_code
    return {"sq_l2": 0, "ip": 1, "neg_ip": 1, "cosine": 2}[metric]


def distances_matrix(Q, mat, metric="sq_l2") -> np.ndarray:
    """[B, n] distances of every query row to every matrix row."""
    Q = N.f32(Q)
    if Q.ndim == 1:
        Q = Q.reshape(1, -1)
    d = Q.shape[1]
    mat = N.f32(mat).reshape(-1, d)
    out = np.empty((Q.shape[0], mat.shape[0]), dtype=np.float32)
    if out.size:
        N.check(N.lib().pk_distances(N.ptr(Q), Q.shape[0], N.ptr(mat), mat.shape[0], d,
                                     _metric_code(metric), N.ptr(out), 0))
    return out


def _one(q, mat, code):
    q = N.f32(q).reshape(-1)
    mat = N.f32(mat).reshape(-1, q.shape[0])
    out = np.empty(mat.shape[0], dtype=np.float32)
    if mat.shape[0]:
        N.check(N.lib().pk_distances(N.ptr(q), 1, N.ptr(mat), mat.shape[0], q.shape[0], code,
                                     N.ptr(out), 0))
    return out


def sq_l2(q, mat) -> np.ndarray:
    """ref/kernels.py:73-83."""
    return _one(q, mat, 0)


def neg_ip(q, mat) -> np.ndarray:
    """ref/kernels.py:86-95."""
    return _one(q, mat, 1)


def cosine(q, mat) -> np.ndarray:
    """ref/kernels.py:98-113."""
    return _one(q, mat, 2)


def kmeans_assign(x, cents):
    """ref/kernels.py:116-135: (labels i64[n], dists f64[n])."""
    x = N.f32(x)
    cents = N.f32(cents).reshape(-1, x.shape[1])
    n = x.shape[0]
    labels = np.zeros(n, dtype=np.int64)
    dists = np.zeros(n, dtype=np.float64)
    if n:
        N.check(N.lib().pk_kmeans_assign(N.ptr(x), n, N.ptr(cents), cents.shape[0], x.shape[1],
                                         N.ptr(labels), N.ptr(dists), 0))
    return labels, dists


BACKENDS = {"cuda": {"sq_l2": sq_l2, "neg_ip": neg_ip, "cosine": cosine, "kmeans_assign": kmeans_assign}}
ACTIVE_BACKEND = "cuda"


def batch_distances(q, mat, metric) -> np.ndarray:
    """ref/core.py:98-109 (no validation; cosine needs non-zero q)."""
    from .core import Metric, UsageError

    mat = np.asarray(mat)
    if mat.shape[0] == 0:
        return np.empty(0, dtype=np.float32)
    if metric is Metric.COSINE:
        qn = float(np.dot(q, q))
        if qn == 0.0:
            raise UsageError("cosine distance requires non-zero vectors")
    return _one(q, mat, _metric_code(metric))


def distance(a, b, metric) -> float:
    """ref/core.py:89-95."""
    from .core import UsageError

    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    if a.shape != b.shape:
        raise UsageError(f"dimension mismatch: {a.shape} vs {b.shape}")
    if not (np.all(np.isfinite(a)) and np.all(np.isfinite(b))):
        raise UsageError("vector contains NaN or Inf")
    return float(batch_distances(a, b[None, :], metric)[0])


def centroid(vectors) -> np.ndarray:
    """ref/core.py:112-117: fp64 row-order mean -> float32 (device)."""
    from .core import UsageError

    mat = N.f32(vectors)
    if mat.ndim == 1:
        mat = mat.reshape(1, -1)
    if len(mat) == 0:
        raise UsageError("centroid of empty vector list")
    out = np.empty(mat.shape[1], dtype=np.float32)
    N.check(N.lib().pk_centroid(N.ptr(mat), mat.shape[0], mat.shape[1], N.ptr(out), 0))
    return out


def deviation(vectors, center, metric) -> float:
    """ref/core.py:120-134: mean member distance in length units."""
    from .core import Metric, UsageError

    mat = N.f32(vectors)
    if len(mat) == 0:
        raise UsageError("deviation of empty vector list")
    if metric is Metric.COSINE:
        d = batch_distances(center, mat, metric)
        return float(np.mean(np.maximum(d, 0.0)))
    d = sq_l2(center, mat)
    return float(np.mean(np.sqrt(np.maximum(d, 0.0))))
