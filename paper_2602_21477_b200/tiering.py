"""Cluster tier bookkeeping (ref/tiering.py:175-448), device-native.

In the reference a simulated accelerator holds snapshots of hot clusters and
a host executor scans the rest; the merged result equals a single-tier scan of
each cluster.  Here every posting list already
lives in the device arena (``DeviceIndex``) and is appended in place, so the
hotset is "all lists" and inserts never need a buffer flush.  The decayed
access frequencies (ref/tiering.py:210-218) and ``metrics()`` are kept so the
store's observable counters have the reference's meaning.

With ``StoreConfig(accelerator="native")`` the cold tier is on: clusters
outside the budgeted hotset live in pinned host memory and are streamed to
HBM when probed, admissions copy on a side stream (TierManager below).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

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


@dataclass
class ResidentCopy:
    """ref/tiering.py:150-154: an HBM copy of a cluster (here the device list
    itself; ``nbytes`` is the budget charge of the admission)."""

    handle: int
    ids: np.ndarray
    nbytes: int


class TierManager:
    """Hotset selection and residency (ref/tiering.py:175-448).

    ``native=False`` (accelerator "none" / "simulated"): every posting list is
    HBM-resident -- 180 GB holds configs[1]-[4] whole -- so the hotset is all
    lists and inserts append in place.  ``native=True`` (accelerator
    "native", configs[4]): the device index runs its cold tier -- lists live
    in pinned host memory, HBM holds the hotset -- and this class is the
    reference's policy verbatim: decayed access frequency (half-life
    ``decay_half_life``), greedy admission by (-frequency, cid) under
    ``budget_bytes``, eviction hysteresis 1.2, run every ``hotset_interval``
    operations by the store.  Admissions copy on a side stream and switch when
    complete; a search scans a cold or in-flight list from a staged copy, so
    results never depend on residency (ref/tiering.py:294-328).
    """

    def __init__(self, store, index, budget_bytes: int = 64 << 20, b_insert: int = 128,
                 decay_half_life: int = 10000, slack_fraction: float = 0.25,
                 hysteresis: float = 1.2, native: bool = False):
        self.store = store
        self.index = index
        self.budget_bytes = budget_bytes
        self.b_insert = b_insert
        self.decay_half_life = decay_half_life
        self.slack_fraction = slack_fraction
        self.hysteresis = hysteresis
        self.native = native
        self.freq: dict[int, tuple[float, int]] = {}
        self.clock = 0
        self._hot: set[int] = set()
        self.resident_bytes = 0
        self.flush_count = 0
        self.aborted = 0
        self._fail_next = False
        self.migration_us: list[float] = []

    # --- frequency tracking (ref/tiering.py:210-218) ---
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
        if not self.native:
            return set(self.store.clusters)
        return set(self._hot)

    # --- hotset (ref/tiering.py:222-262) ---
    def hotset_update(self) -> list[tuple[str, int]]:
        if not self.native:
            return []
        clusters = self.store.clusters
        self._hot &= set(clusters)  # retired clusters left with their device copies
        live = [cid for cid, cl in clusters.items() if cl.size > 0]
        # decayed_freq per cluster, the same float expression in the same
        # order (one evaluation each); ranking (-freq, cid) by one lexsort
        clock, hl, get = self.clock, self.decay_half_life, self.freq.get
        fl = []
        for c in live:
            value, last = get(c, (0.0, clock))
            fl.append(value * (0.5 ** ((clock - last) / hl)))
        freq = dict(zip(live, fl))
        actions: list[tuple[str, int]] = []
        target: list[int] = []
        if live:
            cid_a = np.fromiter(live, dtype=np.int64, count=len(live))
            f_a = np.fromiter(fl, dtype=np.float64, count=len(live))
            nb_a = np.fromiter((clusters[c].nbytes for c in live), dtype=np.int64, count=len(live))
            order = np.lexsort((cid_a, -f_a))
            keep = order[(nb_a[order] > 0) & (f_a[order] > 0.0)]
            # greedy under the budget in rank order: the whole prefix that
            # fits at once, then the rest one by one (a later, smaller
            # cluster may still fit)
            cum = np.cumsum(nb_a[keep])
            n_fit = int(np.searchsorted(cum, self.budget_bytes, side="right"))
            target = cid_a[keep[:n_fit]].tolist()
            used = int(cum[n_fit - 1]) if n_fit else 0
            budget = self.budget_bytes
            for cid, nb in zip(cid_a[keep[n_fit:]].tolist(), nb_a[keep[n_fit:]].tolist()):
                if used + nb <= budget:
                    target.append(cid)
                    used += nb
        target_set = set(target)
        # the displacers (admitted now, not hot before) are the same for every
        # hot cluster examined below: retained clusters are already hot
        displacers = target_set - self._hot
        hottest = max((freq[c] for c in displacers), default=None)
        for cid in sorted(self._hot - target_set):
            if hottest is not None:
                fc = freq[cid] if cid in freq else self.decayed_freq(cid)
                if hottest < self.hysteresis * fc:
                    target_set.add(cid)
                    continue
            actions.append(("evict", cid))
            self._evict(cid)
        for cid in sorted(target_set - self._hot):
            actions.append(("admit", cid))
            self._admit(cid)
        return actions

    @property
    def fail_next_alloc(self) -> bool:
        return self._fail_next
    @fail_next_alloc.setter
    def fail_next_alloc(self, v: bool):
        """The reference's fault-injection seam (``accel.fail_next_alloc``,
        ref/tiering.py:101-104): the next admission's HBM allocation fails in
        the device index (pk_debug_fail_next_alloc)."""
        self._fail_next = bool(v)
        if self.native:
            self.index.fail_next_alloc(1 if v else 0)

    def _admit(self, cid: int):
        """Pending -> Allocated -> Copying -> Switching (device side stream);
        an allocation failure aborts the admission (ref/tiering.py:357-361,
        404-416): the list stays cold with every item, searches unaffected."""
        cl = self.store.clusters[cid]
        nbytes = int(cl.size * cl.dimension * 4 * (1 + self.slack_fraction))
        try:
            self.index.set_resident(cid, True)
        except AcceleratorError:
            self._fail_next = False
            self.aborted += 1
            return
        self._fail_next = False
        cl.resident = ResidentCopy(cid, cl.member_ids.copy(), nbytes)
        cl.buffer_pending = 0
        self.resident_bytes += nbytes
        self._hot.add(cid)

    def _evict(self, cid: int):
        self._hot.discard(cid)
        cl = self.store.clusters.get(cid)
        if cl is None or cl.resident is None:
            return
        self.index.set_resident(cid, False)
        self.resident_bytes -= cl.resident.nbytes
        cl.resident = None
        cl.buffer = []

    # --- insertion path (ref/tiering.py:280-290) ---
    def buffered_insert(self, cid: int, item_id: int, vector) -> str:
        """The device list (and the host copy of a tiered index) is appended
        in place, so there is no insertion buffer to flush."""
        self.store.add_member(cid, item_id, vector)
        cl = self.store.clusters[cid]
        if self.native and cl.resident is None:
            return "DirectHost"
        self._count_flushes(cl, 1)
        return "DeviceInPlace"

    def buffered_insert_many(self, cid: int, item_ids: np.ndarray, vectors: np.ndarray):
        """buffered_insert of consecutive items of one cluster."""
        self.store.add_members(cid, item_ids, vectors)
        cl = self.store.clusters[cid]
        if not (self.native and cl.resident is None):
            self._count_flushes(cl, len(item_ids))

    def buffered_insert_batch(self, cids: np.ndarray, item_ids: np.ndarray, vectors: np.ndarray):
        """buffered_insert of a run of items (per cluster in batch order): one
        queued device append for the run, the host mirrors per cluster."""
        for cid, n in self.store.add_members_batch(cids, item_ids, vectors):
            cl = self.store.clusters[cid]
            if not (self.native and cl.resident is None):
                self._count_flushes(cl, n)

    def _count_flushes(self, cl, n: int):
        """``buffer_flush_count`` keeps the reference's meaning on the native
        tier: the reference buffers inserts into a resident cluster and flushes
        them to the device every ``b_insert`` (ref/tiering.py:280-290); here
        the rows reach HBM in place, and a flush is counted at each
        ``b_insert``-th insert into a resident list."""
        if not self.native:
            return
        cl.buffer_pending = getattr(cl, "buffer_pending", 0) + n
        while cl.buffer_pending >= self.b_insert:
            cl.buffer_pending -= self.b_insert
            self.flush_count += 1

    # --- splitting (ref/tiering.py:420-434) ---
    def split_offload(self, cid: int):
        cl = self.store.clusters[cid]
        was_resident = self.native and cl.resident is not None
        if was_resident:
            self._evict(cid)
        outcome = self.store.split_cluster(cid)
        parent_freq = self.decayed_freq(cid)
        self.freq.pop(cid, None)
        for child in outcome.children:
            self.freq[child] = (parent_freq / max(len(outcome.children), 1), self.clock)
        if was_resident:
            self.hotset_update()
        return outcome

    # --- metrics (ref/tiering.py:438-448) ---
    def metrics(self) -> dict:
        live = [c for c in self.store.clusters.values() if c.size > 0]
        if self.native:
            resident = sum(1 for c in live if c.resident is not None)
            ratio = resident / len(live) if live else 0.0
        else:
            ratio = 1.0 if live else 0.0
        out = {
            "residency_ratio": ratio,
            "buffer_flush_count": self.flush_count,
            "aborted_admissions": self.aborted,
            "migration_us": list(self.migration_us),
            "resident_bytes": self.resident_bytes if self.native else sum(c.nbytes for c in live),
            "host_us": 0.0,
            "accel_us": 0.0,
            "device_bytes": self.index.nbytes(),
        }
        if self.native:
            out.update({f"tier_{k}": v for k, v in self.index.tier_stats().items()})
        return out
