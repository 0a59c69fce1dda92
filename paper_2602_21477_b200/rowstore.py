"""Slots of the device index's HBM row store (pk_rows_put / pk_agent_read).

The agent path's policy scans small vector sets over and over -- the cache's
pool rows (ref/cache.py:162-221), the L1 centroids, staged items
(ref/engine.py:353-363) and the FSM states (ref/fsm.py:62-90).  Here each of
those rows gets a slot in one HBM row store when it is created and keeps it
until it is dropped, so a search names the rows it reads by slot and ships only
its query.  New rows are queued and uploaded with the next device call
(``take_puts``); the latest write to a slot wins, and a slot freed before its
upload never crosses PCIe.
"""

from __future__ import annotations

import threading

import numpy as np


class RowStore:
    def __init__(self, index, dimension: int):
        self.index = index
        self.dimension = dimension
        self._free: list[int] = []
        self._next = 0
        self._pend: dict[int, np.ndarray] = {}
        # held across take_puts + the device call that applies them, so two
        # agents' searches cannot read a slot before its row is uploaded
        self.lock = threading.RLock()

    def alloc(self, vec) -> int:
        with self.lock:
            s = self._free.pop() if self._free else self._next
            if s == self._next:
                self._next += 1
            self._pend[s] = np.array(vec, dtype=np.float32, copy=True).reshape(self.dimension)
            return s

    def put(self, slot: int, vec):
        """Overwrite a live slot's row (an L1 centroid after its cluster changed)."""
        with self.lock:
            self._pend[int(slot)] = np.array(vec, dtype=np.float32, copy=True).reshape(self.dimension)

    def free(self, slot: int):
        if slot < 0:
            return
        with self.lock:
            self._pend.pop(slot, None)
            self._free.append(slot)

    def free_many(self, slots):
        with self.lock:
            for s in np.asarray(slots).tolist():
                if s >= 0:
                    self._pend.pop(s, None)
                    self._free.append(s)

    def reserve(self, extra: int):
        """Device capacity for ``extra`` more slots than are allocated now."""
        self._reserved = max(getattr(self, "_reserved", 0), self._next) + int(extra)
        self.index.rows_reserve(self._reserved)

    @property
    def live(self) -> int:
        return self._next - len(self._free)

    def take_puts(self):
        """(slots i32[n], rows f32[n, d]) queued since the last call, cleared."""
        if not self._pend:
            return None, None
        slots = np.fromiter(self._pend.keys(), dtype=np.int32, count=len(self._pend))
        rows = np.stack(list(self._pend.values()))
        self._pend.clear()
        return slots, rows

    def flush(self):
        with self.lock:
            slots, rows = self.take_puts()
            if slots is not None:
                self.index.rows_put(slots, rows)
