"""NativeAccelerator: the reference's executor plugin protocol on the B200
(layer 2; protocol of ``SimulatedAccelerator``,
ref/tiering.py:85-147).

For a maintainer who keeps the reference's own ``TierManager`` and swaps only
the executor (``StoreConfig(accelerator=...)`` -> this class), every call
maps onto the device index of this package:

  alloc(nbytes)               -> a fresh empty posting list (the handle)
  upload(h, mat, ids, local)  -> appended rows (ref upload appends, tiering.py:112-123)
  release(h, nbytes)          -> list retired, HBM range freed
  scan(h, q, metric)          -> (ids, distances) of the snapshot in row order,
                                 reference arithmetic on the device
                                 (pk_scan_lists; batch_distances semantics)
  kmeans(mat, k, rng, delta)  -> kmeans_split_points on the device, consuming
                                 ``rng`` exactly like the reference (F6)

plus the observable attributes the reference and its tests read:
``allocated_bytes``, ``call_log``, ``simulated_us`` (cost-model accounting,
unchanged), ``fail_next_alloc`` / ``fail_next_scan`` and ``_mem[handle] ->
(mat, ids)`` (read back from the device, tiering.py:387-390).  Errors raise
``AcceleratorError`` as the protocol expects -- this package's, or the host's own
class when given (``error_type``: a maintainer plugging this executor into the
reference's ``TierManager`` passes ``agentmem.tiering.AcceleratorError``, the
type its host-fallback handlers catch, ref/tiering.py:308-311, 357-361).
"""

from __future__ import annotations

import numpy as np

from .clusters import kmeans_split_points
from .core import AcceleratorError, Metric
from .index import DeviceIndex
from .tiering import CostModel


class _MemView:
    """``accel._mem[handle] -> (mat f32[n, d], ids i64[n])`` read from HBM."""

    def __init__(self, acc: "NativeAccelerator"):
        self._acc = acc

    def __contains__(self, handle) -> bool:
        return handle in self._acc._live

    def __getitem__(self, handle):
        if handle not in self._acc._live:
            raise KeyError(handle)
        return self._acc._read(handle)

    def get(self, handle, default=None):
        return self[handle] if handle in self._acc._live else default

    def pop(self, handle, default=None):
        if handle not in self._acc._live:
            return default
        out = self._acc._read(handle)
        self._acc._drop(handle)
        return out

    def __len__(self):
        return len(self._acc._live)


class NativeAccelerator:
    kind = "accelerator"
    capabilities = frozenset({"scan", "kmeans"})

    def __init__(self, model: CostModel | None = None, dimension: int | None = None,
                 metric: Metric = Metric.SQUARED_EUCLIDEAN, device: int = 0,
                 error_type: type = AcceleratorError):
        self.model = model or CostModel()
        self.call_log: list[tuple] = []
        self.simulated_us = 0.0
        self.allocated_bytes = 0
        self.fail_next_alloc = False
        self.fail_next_scan = False
        self._metric = _as_metric(metric)
        self._err = error_type
        self._device = device
        self._dimension = dimension
        self._index: DeviceIndex | None = None
        self._next_handle = 0
        self._live: dict[int, int] = {}  # handle -> rows held
        self._cid: dict[int, int] = {}   # handle -> list id in the shared device index
        self._mem = _MemView(self)

    # ---- device index: one per (device, dimension, metric), shared by every
    # executor of this process (a TierManager per cluster store, as the
    # reference's tests build thousands of, must not each pay an index
    # creation); created at the first upload -- the dimension is the first
    # matrix's width unless given ---------------------------------------------
    _shared: dict = {}
    _next_cid = 0

    def _ix(self, d: int) -> DeviceIndex:
        if self._index is None:
            self._dimension = self._dimension or d
            key = (self._device, self._dimension, self._metric)
            ix = NativeAccelerator._shared.get(key)
            if ix is None:
                ix = DeviceIndex(self._dimension, self._metric.wire_code, self._device)
                NativeAccelerator._shared[key] = ix
            self._index = ix
        if d != self._dimension:
            raise self._err(f"dimension mismatch: {d} vs {self._dimension}")
        return self._index

    def _read(self, handle):
        n = self._live[handle]
        if n == 0 or self._index is None:
            return (np.empty((0, 0), dtype=np.float32), np.empty(0, dtype=np.int64))
        rows, ids = self._index.read(self._cid[handle])
        return rows, ids

    def _drop(self, handle):
        cid = self._cid.pop(handle, None)
        if self._live.pop(handle, 0) > 0 and self._index is not None and cid is not None:
            self._index.retire(cid)

    # ---- protocol (ref/tiering.py:101-147) -------------------------------
    def alloc(self, nbytes: int) -> int:
        if self.fail_next_alloc:
            self.fail_next_alloc = False
            raise self._err("allocation failed")
        handle = self._next_handle
        self._next_handle += 1
        self._live[handle] = 0
        self.allocated_bytes += nbytes
        self.simulated_us += self.model.alloc_us
        self.call_log.append(("alloc", handle, nbytes))
        return handle

    def upload(self, handle: int, mat: np.ndarray, ids: np.ndarray, tier_local: bool):
        if handle not in self._live:
            raise self._err(f"unknown handle {handle}")
        mat = np.ascontiguousarray(mat, dtype=np.float32)
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        if len(ids):
            ix = self._ix(mat.shape[1])
            if self._live[handle] == 0:  # first rows: the list comes into existence
                cid = NativeAccelerator._next_cid
                NativeAccelerator._next_cid += 1
                ix.create_list(cid, 0, mat, ids)
                self._cid[handle] = cid
            else:
                ix.append(self._cid[handle], mat, ids)
            self._live[handle] += len(ids)
        kb = (self._live[handle] * (self._dimension or 0) * 4) / 1024.0
        rate = self.model.tier_local_per_kb_us if tier_local else self.model.cross_tier_per_kb_us
        self.simulated_us += kb * rate
        self.call_log.append(("upload", handle, len(ids), tier_local))

    def release(self, handle: int, nbytes: int):
        if handle in self._live:
            self._drop(handle)
        self.allocated_bytes -= nbytes
        self.call_log.append(("release", handle))

    def scan(self, handle: int, q: np.ndarray, metric: Metric):
        if self.fail_next_scan:
            self.fail_next_scan = False
            raise self._err("device scan failed")
        if handle not in self._live:
            raise self._err(f"unknown handle {handle}")
        n = self._live[handle]
        self.call_log.append(("scan", handle, n))
        self.simulated_us += self.model.accel_scan_us(n)
        if n == 0:
            return np.empty(0, dtype=np.int64), np.empty(0, dtype=np.float32)
        if _as_metric(metric) is not self._metric:
            raise self._err(f"index built for {self._metric}, scan asked {metric}")
        ids, dists, _ = self._index.scan_lists(np.asarray(q, dtype=np.float32), [self._cid[handle]], n)
        return ids, dists

    def kmeans(self, mat, k, rng, base_delta):
        self.call_log.append(("kmeans", len(mat), k))
        self.simulated_us += self.model.accel_scan_us(len(mat)) * k
        return kmeans_split_points(np.ascontiguousarray(mat, dtype=np.float32), k, rng, base_delta,
                                   device=self._device)

    def close(self):
        """Release every list this executor still holds (the shared device
        index stays for the other executors)."""
        for handle in list(self._live):
            self._drop(handle)
        self._index = None

    def __del__(self):  # pragma: no cover - garbage collection order
        try:
            self.close()
        except Exception:
            pass


def _as_metric(m) -> Metric:
    """This package's Metric for a Metric of either package (the reference's
    TierManager passes its own enum members; same values)."""
    return m if isinstance(m, Metric) else Metric(getattr(m, "value", m))
