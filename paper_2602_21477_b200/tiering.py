"""Cluster tier bookkeeping (ref/tiering.py:175-448), device-native.

In the reference a simulated accelerator holds snapshots of hot clusters and
a host executor scans the rest; the merged result equals a single-tier scan of
each cluster.  Here every posting list already
lives in the device arena (``DeviceIndex``) and is appended in place, so the
hotset is "all lists" and inserts never need a buffer flush.  The decayed
access frequencies (ref/tiering.py:210-218) and ``metrics()`` are kept so the
store's observable counters have the reference's meaning.

The pinned-host cold tier (clusters beyond ``budget_bytes`` streamed on a side
stream) is the next step of this module ("What comes next").
"""

from __future__ import annotations

from dataclasses import dataclass

from .core import AcceleratorError  # noqa: F401  (re-exported name)


@dataclass
class CostModel:
    """Kept for API compatibility (ref/tiering.py:33-48); not used for timing."""

    host_per_vector_us: float = 0.5
    accel_launch_us: float = 64.0
    accel_per_vector_us: float = 0.0
    cross_tier_per_kb_us: float = 1.0
    tier_local_per_kb_us: float = 0.05
    alloc_us: float = 10.0

    def host_scan_us(self, n: int) -> float:
        return self.host_per_vector_us * n

    def accel_scan_us(self, n: int) -> float:
        return self.accel_launch_us + self.accel_per_vector_us * n


def derive_b_insert(model: CostModel, max_n: int = 1 << 20) -> int:
    """ref/tiering.py:51-62."""
    n, lo, hi = 0, 0, max_n
    while lo <= hi:
        mid = (lo + hi) // 2
        if model.host_scan_us(mid) <= model.accel_scan_us(mid):
            n = mid
            lo = mid + 1
        else:
            hi = mid - 1
    return n


class TierManager:
    def __init__(self, store, index, budget_bytes: int = 64 << 20, b_insert: int = 128,
                 decay_half_life: int = 10000, slack_fraction: float = 0.25):
        self.store = store
        self.index = index
        self.budget_bytes = budget_bytes
        self.b_insert = b_insert
        self.decay_half_life = decay_half_life
        self.slack_fraction = slack_fraction
        self.freq: dict[int, tuple[float, int]] = {}
        self.clock = 0
        self.flush_count = 0
        self.migration_us: list[float] = []

    def record_access(self, cid: int):
        self.clock += 1
        value, last = self.freq.get(cid, (0.0, self.clock))
        decay = 0.5 ** ((self.clock - last) / self.decay_half_life)
        self.freq[cid] = (value * decay + 1.0, self.clock)

    def decayed_freq(self, cid: int) -> float:
        value, last = self.freq.get(cid, (0.0, self.clock))
        return value * (0.5 ** ((self.clock - last) / self.decay_half_life))

    @property
    def hotset(self) -> set[int]:
        return set(self.store.clusters)

    def hotset_update(self):
        return []

    def buffered_insert(self, cid: int, item_id: int, vector) -> str:
        """ref/tiering.py:280-290: the device list is appended in place."""
        self.store.add_member(cid, item_id, vector)
        return "DeviceInPlace"

    def split_offload(self, cid: int):
        """ref/tiering.py:420-434: split with the device k-means."""
        outcome = self.store.split_cluster(cid)
        parent_freq = self.decayed_freq(cid)
        self.freq.pop(cid, None)
        for child in outcome.children:
            self.freq[child] = (parent_freq / max(len(outcome.children), 1), self.clock)
        return outcome

    def _evict(self, cid: int):
        return None

    def metrics(self) -> dict:
        live = [c for c in self.store.clusters.values() if c.size > 0]
        return {
            "residency_ratio": 1.0 if live else 0.0,
            "buffer_flush_count": self.flush_count,
            "migration_us": list(self.migration_us),
            "resident_bytes": sum(c.nbytes for c in live),
            "host_us": 0.0,
            "accel_us": 0.0,
            "device_bytes": self.index.nbytes(),
        }
