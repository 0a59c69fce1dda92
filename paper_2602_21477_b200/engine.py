"""Public store facade, a drop-in for the reference's ``agentmem.engine``
(ref/engine.py:1-839) on the bare IVF path.

Same classes and signatures (``Store``, ``StoreConfig``, ``SearchResult``,
``SearchStats``, ``OperationBatch``), same validation and error types, same
results.  What changes is underneath: the coarse quantizer, the posting-list
scan, the top-k merge, assignment and centroid maintenance run as sm_100a
kernels over a device-resident index (``DeviceIndex``), and batches of
queries are answered by ONE device pass (``search_batch`` / ``submit_batch``)
instead of one Python loop iteration per (query, cluster).

Two read paths: a batch of bare queries (``agent=None``, or an agent
without a cache, and no staged items in scope) is ONE device pass
(coarse on tcgen05, screened scan, exact re-rank); an agent query with its
multi-level cache (ref/cache.py), staged items (ref/engine.py:353-363) or
early termination (ref/engine.py:376-396) runs the reference's per-query
pipeline with every distance from ONE device pass (pk_agent_read): the FSM
states, every cached pool row and L1 centroid (resident in an HBM row store,
rowstore.RowStore), the staged rows, the reference's coarse graph traversal
and every row of the lists it probes -- then the hint, scan order, stop rules
and _topk are replayed on those values.  The L1 placement chain of a
promotion is one more device call when L0 overflows (pk_l1_place).
"""

from __future__ import annotations

import os
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from . import pnck
from .cache import DEFAULT_KEY, MultiLevelCache
from .clusters import ClusterStore, SplitOutcome, kmeans_split_points
from .fsm import PatternHint, PatternTable
from .concurrency import RWLock, TaskRunner
from .core import (
    STATIC_SCOPE,
    Metric,
    ScopePermissionError,
    UsageError,
    as_matrix,
    as_vector,
)
from .index import DeviceIndex
from .rowstore import RowStore
from .kernels import centroid as vector_mean
from .kernels import deviation as vector_spread
from .tiering import TierManager

SEED_ENV = "PANCAKE_SEED"


@dataclass
class StoreConfig:
    """ref/engine.py:42-100 (every field kept); ``device`` is new."""

    dimension: int
    metric: Metric = Metric.SQUARED_EUCLIDEAN
    seed: int = 0
    split_threshold: int = 4096
    split_target: int = 2048
    maintenance_interval: int = 256
    n_p: int = 16
    l0_capacity: int = 64
    l1_capacity: int = 1024
    kappa: int = 2
    alpha_et: float = 0.7
    window_w: int = 32
    verify_mode: bool = False
    cache_enabled: bool = True
    n_s: int = 8
    d_merge_factor: float = 0.5
    theta_match: float = 0.5
    prefetch_enabled: bool = True
    pattern_enabled: bool = True
    m: int = 16
    ef_search_factor: int = 4
    alpha_ic: float = 6.0
    p_size: int = 32
    coarse_mode: str = "hybrid"
    profiles_enabled: bool = True
    accelerator: str = "simulated"
    budget_bytes: int = 64 << 20
    b_insert: int = 128
    decay_half_life: int = 10000
    slack_fraction: float = 0.25
    hotset_interval: int = 64
    splits_enabled: bool = True
    lazy_maintenance: bool = True
    static_writable_by_agents: bool = False
    default_nprobe: int = 8
    threads: int = 0
    request_window: int = 64
    device: int = 0
    # new: under torch.distributed (one process per GPU, every rank making the
    # same calls) the posting lists are partitioned over the ranks' HBM,
    # agents' lists co-located per rank (sharded.ShardedStoreIndex)
    sharded: bool = False

    def __post_init__(self):
        if not isinstance(self.metric, Metric):  # a name, or another package's Metric member
            self.metric = Metric(getattr(self.metric, "value", self.metric))
        if self.dimension < 1:
            raise UsageError(f"dimension must be >= 1, got {self.dimension}")
        if not 0.0 <= self.alpha_et <= 1.0:
            raise UsageError("alpha_et must lie in [0, 1]")
        if self.split_target >= self.split_threshold:
            raise UsageError("split_target must be below split_threshold")
        if self.coarse_mode not in ("hybrid", "per_agent"):
            raise UsageError(f"unknown coarse_mode {self.coarse_mode!r}")
        if self.accelerator not in ("none", "simulated", "native"):
            raise UsageError(f"unknown accelerator {self.accelerator!r}")


@dataclass
class SearchStats:
    scanned_vectors: int = 0
    coarse_computations: int = 0
    level_reached: str = "L2"
    early_terminated: bool = False


@dataclass
class SearchResult:
    hits: list[tuple[int, float, str]]
    stats: SearchStats
    scan_ids: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int64))

    @property
    def ids(self) -> list[int]:
        return [h[0] for h in self.hits]

    @property
    def distances(self) -> list[float]:
        return [h[1] for h in self.hits]


@dataclass
class OperationBatch:
    kind: str
    agent: str | None
    ops: list

    def __post_init__(self):
        if self.kind not in ("search", "insert", "update", "delete"):
            raise UsageError(f"unknown batch kind {self.kind!r}")


class ScopeCodes:
    """Store-wide scope -> small int interning (ref/pool.py:14-30)."""

    def __init__(self):
        self.code: dict[str, int] = {}
        self.name: list[str] = []

    def intern(self, scope: str) -> int:
        c = self.code.get(scope)
        if c is None:
            c = len(self.name)
            self.code[scope] = c
            self.name.append(scope)
        return c

    def mask_codes(self, scopes) -> np.ndarray:
        return np.asarray(sorted(self.intern(s) for s in scopes), dtype=np.int16)

    def lut(self, scopes):
        """(boolean table over codes, hashable key) of a scope set."""
        codes = tuple(sorted(self.intern(s) for s in scopes))
        t = np.zeros(max(len(self.name), 1) + 1, dtype=bool)
        t[list(codes)] = True
        return t, codes


def profile_reorder(entries, default_order):
    """ref/graph.py:441-451."""
    default_set = set(default_order)
    seen, front = set(), []
    for lid in entries:
        if lid in default_set and lid not in seen:
            front.append(lid)
            seen.add(lid)
    return front + [lid for lid in default_order if lid not in seen]


def profile_order(entries, size: int) -> np.ndarray:
    """``profile_reorder(entries, range(size))`` as index arrays: the profile's
    rows first (first occurrence, rows outside [0, size) skipped), then every
    other row in order -- the per-probed-list scan order of scan_ids, without
    a Python pass over all of the list's rows."""
    if not entries:
        return np.arange(size)
    e = np.asarray(entries, dtype=np.int64)
    e = e[(e >= 0) & (e < size)]
    if len(e) == 0:
        return np.arange(size)
    _, first = np.unique(e, return_index=True)
    front = e[np.sort(first)]
    rest = np.ones(size, dtype=bool)
    rest[front] = False
    return np.concatenate([front, np.flatnonzero(rest)])


def profile_promote(entries, hits, p_size):
    """ref/graph.py:454-463."""
    hit_seen, front = set(), []
    for lid in hits:
        if lid not in hit_seen:
            front.append(lid)
            hit_seen.add(lid)
    return (front + [lid for lid in entries if lid not in hit_seen])[:p_size]


class Store:
    """One memory store: a static scope plus any number of agent scopes."""

    def __init__(self, cfg: StoreConfig):
        self.cfg = cfg
        seed = cfg.seed
        env = os.environ.get(SEED_ENV)
        if env is not None:
            seed = int(env)
        self.seed = seed
        self.rng = np.random.default_rng(np.random.PCG64(seed))
        self.metric = cfg.metric
        self.scope_codes = ScopeCodes()
        if cfg.sharded:
            from .sharded import ShardedStoreIndex

            self.index = ShardedStoreIndex(cfg.dimension, cfg.metric.wire_code, cfg.device)
        else:
            self.index = DeviceIndex(cfg.dimension, cfg.metric.wire_code, cfg.device)
        native_tier = cfg.accelerator == "native"
        if native_tier:  # cold tier: pinned host memory, HBM holds the hotset
            self.index.enable_tier()
        self.clusters = ClusterStore(
            cfg.dimension, cfg.metric, self.rng, self.index, self.scope_codes,
            split_threshold=cfg.split_threshold, split_target=cfg.split_target,
            maintenance_interval=cfg.maintenance_interval, m=cfg.m,
            ef_search_factor=cfg.ef_search_factor, alpha_ic=cfg.alpha_ic,
        )
        self.graph = self.clusters.graph
        # HBM rows of the agent policy's small vector sets (pools, L1
        # centroids, staged items, FSM states), one slot each
        self.rows = RowStore(self.index, cfg.dimension)
        self.clusters.rows = self.rows
        self._drows: dict[str, list] = {}  # per agent: D rows of its request sequence
        self._qrow_memo: dict = {}  # per agent: the last hinted query's D row
        self._list_cap = 2 * cfg.split_target  # rows per probed list the agent pass reserves
        self._tiered_native = native_tier
        self._lists_pf = None  # an agent search batch's prefetched lists (_prefetch_lists)
        self.runner = TaskRunner(cfg.threads)
        self.tier = TierManager(self.clusters, self.index, budget_bytes=cfg.budget_bytes,
                                b_insert=cfg.b_insert, decay_half_life=cfg.decay_half_life,
                                slack_fraction=cfg.slack_fraction, native=native_tier)
        self.agents: set[str] = set()
        self.caches: dict[str, MultiLevelCache] = {}
        self.patterns: dict[str, PatternTable] = {}
        self._prefetch_inflight: set = set()
        self._match_memo: dict = {}
        self.sequences: dict[str, list[np.ndarray]] = {}
        self.payloads: dict[int, bytes] = {}
        self._next_item_id = 0
        self._op_count = 0
        self._lock = RWLock()
        self._agent_locks: dict[str, threading.RLock] = {}
        self._ingest_lock = threading.RLock()
        self.clusters.register_scope(STATIC_SCOPE)
        self.scope_codes.intern(STATIC_SCOPE)

    # --- lifecycle --------------------------------------------------------
    @classmethod
    def create(cls, cfg: StoreConfig) -> "Store":
        return cls(cfg)

    def close(self):
        self.runner.shutdown()
        self.index.close()

    def _centroid_of(self, cid: int) -> np.ndarray:
        return self.clusters.clusters[cid].centroid

    # --- scopes -----------------------------------------------------------
    def register_agent(self, agent_id: str) -> str:
        """ref/engine.py:211-241."""
        if agent_id == STATIC_SCOPE:
            raise UsageError(f"{STATIC_SCOPE!r} is reserved for the shared base scope")
        if agent_id in self.agents:
            raise UsageError(f"agent {agent_id!r} already registered")
        self.clusters.register_scope(agent_id)
        self.scope_codes.intern(agent_id)
        self.agents.add(agent_id)
        c = self.cfg
        self.caches[agent_id] = MultiLevelCache(
            agent_id, c.dimension, self.metric, self.scope_codes, n_p=c.n_p,
            l0_capacity=c.l0_capacity, l1_capacity=c.l1_capacity, kappa=c.kappa,
            alpha_et=c.alpha_et, window_w=c.window_w, verify_mode=c.verify_mode, rows=self.rows)
        self.patterns[agent_id] = PatternTable(n_p=c.n_p, n_s=c.n_s, metric=self.metric,
                                               theta_match=c.theta_match,
                                               d_merge_factor=c.d_merge_factor, rows=self.rows)
        self.sequences[agent_id] = []
        self._drows[agent_id] = []
        self._agent_locks[agent_id] = threading.RLock()
        # the agent's bound in the HBM row store -- n_p L0 pools, n_p L1 pools
        # and n_p patterns of n_s states -- reserved now, not grown mid-stream
        self.rows.reserve(c.n_p * (c.l0_capacity + c.l1_capacity + c.n_s) + 64)
        return agent_id

    def unregister_agent(self, agent_id: str):
        if agent_id not in self.agents:
            raise UsageError(f"unknown agent {agent_id!r}")
        for cid in list(self.clusters.scope_clusters(agent_id)):
            self.tier._evict(cid)
            self.clusters.retire_cluster(cid)
        for item_id in list(self.clusters.staged.get(agent_id, {})):
            self.clusters.unstage(agent_id, item_id)
            self.payloads.pop(item_id, None)
        self.agents.discard(agent_id)
        cache = self.caches.pop(agent_id, None)
        if cache is not None:
            for entry in cache.l0.values():
                entry.pool.release()
            for cl in cache.l1:
                cl.release(self.rows)
        table = self.patterns.pop(agent_id, None)
        if table is not None:
            for _, sl in table._slots:
                self.rows.free_many(sl)
        del self.sequences[agent_id]
        self._drows.pop(agent_id, None)
        del self._agent_locks[agent_id]

    def registered_scopes(self) -> list[str]:
        return list(self.clusters.by_scope)

    def _serialized(self, agent):
        if agent is None:
            return self._ingest_lock
        return self._agent_locks[agent]

    def _check_scopes(self, scopes) -> set[str]:
        out = set(scopes)
        if not out:
            raise UsageError("scope set must be non-empty")
        for sc in out:
            if sc not in self.clusters.by_scope:
                raise UsageError(f"unknown scope {sc!r}")
        return out

    def _check_writable(self, agent, scope: str):
        if scope not in self.clusters.by_scope:
            raise UsageError(f"unknown scope {scope!r}")
        if agent is None or scope == agent:
            return
        if scope == STATIC_SCOPE and self.cfg.static_writable_by_agents:
            return
        raise ScopePermissionError(f"agent {agent!r} may not write scope {scope!r}")

    def _agent_path(self, agent, scopes, no_cache=False, k: int = 1) -> bool:
        """True when a query needs the per-query pipeline: an agent cache in
        use, pattern hints (prefetch), staged (cache-owned) items in a
        searched scope, or k above the batched device top-k (KKMAX): that
        pipeline ranks every probed row (pk_scan_lists) for any k."""
        if k > N.KKMAX:
            return True
        if agent is not None and agent in self.caches:
            if self.cfg.cache_enabled and not no_cache:
                return True
            if self.cfg.pattern_enabled:  # hints drive prefetch (ref/engine.py:498-501)
                return True
        return any(self.clusters.staged.get(sc) for sc in scopes)

    # --- search -----------------------------------------------------------
    def search(self, agent, scopes, q, k: int, nprobe: int | None = None, _internal: bool = False,
               _no_cache: bool = False) -> SearchResult:
        """ref/engine.py:287-317."""
        if k < 1:
            raise UsageError("k must be >= 1")
        scopes = self._check_scopes(scopes)
        if agent is not None and agent not in self.agents:
            raise UsageError(f"unknown agent {agent!r}")
        q = as_vector(q, self.cfg.dimension)
        nprobe = nprobe if nprobe is not None else self.cfg.default_nprobe
        if nprobe < 1:
            raise UsageError("nprobe must be >= 1")
        with self._serialized(agent):
            self._lock.acquire_read()
            try:
                if self._agent_path(agent, scopes, _no_cache, k):
                    result, hint, extended = self._search_read_phase(agent, scopes, q, k, nprobe,
                                                                     _internal, _no_cache)
                else:
                    result = self._search_read_phase_batch(agent, scopes, q[None, :], k, nprobe,
                                                           want_scan_ids=True)[0]
                    hint, extended = PatternHint(), None
            finally:
                self._lock.release_read()
            if agent is not None:
                self._search_side_effects(agent, q, k, hint, result, extended, _internal)
            self._tick()
            return result

    def search_batch(self, agent, scopes, Q, k: int, nprobe: int | None = None,
                     want_scan_ids: bool = False) -> list[SearchResult]:
        """B queries with the same (agent, scopes, k, nprobe) in one device
        pass; equal to B calls of ``search`` (``scan_ids`` only on request)."""
        if k < 1:
            raise UsageError("k must be >= 1")
        scopes = self._check_scopes(scopes)
        if agent is not None and agent not in self.agents:
            raise UsageError(f"unknown agent {agent!r}")
        Q = as_matrix(Q, self.cfg.dimension)
        nprobe = nprobe if nprobe is not None else self.cfg.default_nprobe
        if nprobe < 1:
            raise UsageError("nprobe must be >= 1")
        if self._agent_path(agent, scopes, k=k) or (agent is not None and self.cfg.profiles_enabled):
            # per-query pipeline, B calls of search(): with agent profiles on,
            # each query's scan order depends on the profile updates of the
            # queries before it (ref/engine.py:488-496), so they cannot share
            # one read phase.  What they can share is the device half that
            # no side effect changes: the coarse traversal and the probed
            # lists' rows of every query, in one pass (used while the lists,
            # centroids and graph are unchanged)
            if Q.shape[0] > 1 and self._agent_path(agent, scopes, k=k):
                self._prefetch_lists(scopes, Q, k, nprobe)
            try:
                return [self.search(agent, scopes, Q[b], k, nprobe) for b in range(Q.shape[0])]
            finally:
                self._lists_pf = None
        with self._serialized(agent):
            self._lock.acquire_read()
            try:
                results = self._search_read_phase_batch(agent, scopes, Q, k, nprobe, want_scan_ids)
            finally:
                self._lock.release_read()
            for b, res in enumerate(results):
                if agent is not None:
                    self._search_side_effects(agent, Q[b], k, PatternHint(), res, None, False)
                self._tick()
            return results

    def _prefetch_lists(self, scopes, Q, k, nprobe):
        """pk_agent_lists for the queries of an agent's search batch: what
        _search_read_phase's agent_read would compute for their lists, keyed
        by the query bytes and the plan, stamped with the list version."""
        self._lists_pf = None
        if self._tiered_native or not hasattr(self.index, "agent_lists") or not self.clusters.clusters:
            return
        self._lock.acquire_read()
        try:
            eff_nprobe, ef, mode = self._coarse_plan(k, nprobe)
            in_scope = sum(len(self.clusters.by_scope[s]) for s in scopes)
            dev_nprobe = max(1, min(eff_nprobe, in_scope))
            codes = [self.scope_codes.intern(s) for s in sorted(scopes)]
            self.graph.upload()
            ver, outs = self.index.agent_lists(Q, codes, dev_nprobe, ef, mode, dev_nprobe * self._list_cap)
            plan = (tuple(codes), dev_nprobe, ef, mode)
            self._lists_pf = (ver, plan, {Q[b].tobytes(): o for b, o in enumerate(outs) if o is not None})
        finally:
            self._lock.release_read()

    def _prefetched_lists(self, q, plan):
        pf = self._lists_pf
        if pf is None or pf[1] != plan:
            return None
        lists = pf[2].get(q.tobytes())
        if lists is None or pf[0] != self.index.list_version():
            return None
        return lists

    def _coarse_plan(self, k, nprobe):
        """(eff_nprobe, ef, mode) of the coarse traversal (ref/engine.py:365-373,
        ref/graph.py:338-340): the exhaustive edge probes every list with
        ef = eff_nprobe * ef_search_factor."""
        eff_nprobe, ef_search = nprobe, None
        if k >= self.clusters.live_count():
            eff_nprobe = max(nprobe, len(self.clusters.clusters) or 1)
            ef_search = eff_nprobe * self.cfg.ef_search_factor
        mode = 1 if self.cfg.coarse_mode == "per_agent" else 0
        return eff_nprobe, min(self.graph.ef_for(eff_nprobe, ef_search), 1 << 30), mode

    def _search_read_phase_batch(self, agent, scopes, Q, k, nprobe, want_scan_ids):
        """Store._search_read_phase (ref/engine.py:319-404) for a batch on the
        bare path: the reference's graph traversal as the coarse stage (any
        ef), merged scan of every probed list and _topk (ref/engine.py:406-426)
        in one device pass (pk_search_graph)."""
        B = Q.shape[0]
        eff_nprobe, ef, mode = self._coarse_plan(k, nprobe)
        in_scope = sum(len(self.clusters.by_scope[s]) for s in scopes)
        dev_nprobe = max(1, min(eff_nprobe, in_scope))
        if dev_nprobe > N.NPROBE_MAX or not self.clusters.clusters:
            # more probed lists than the fused pass scans (or no lists at
            # all): the per-query pipeline serves it
            return [self._search_read_phase(agent, scopes, Q[b], k, nprobe, True, True)[0]
                    for b in range(B)]
        codes = [self.scope_codes.intern(s) for s in sorted(scopes)]
        self.graph.upload()
        out, coarse = self.index.search_graph(Q, codes, dev_nprobe, k, ef, mode, want_probe=True)
        results = []
        clusters = self.clusters.clusters
        for b in range(B):
            n = int(out.counts[b])
            ids = out.ids[b, :n].tolist()
            dd = out.dists[b, :n].tolist()
            cs = out.cids[b, :n].tolist()
            hits = [(ids[i], dd[i], clusters[cs[i]].scope) for i in range(n)]
            stats = SearchStats(scanned_vectors=int(out.scanned[b]),
                                coarse_computations=int(coarse[b]),
                                level_reached="L2", early_terminated=False)
            probe = [c for c in out.probe[b].tolist() if c >= 0]
            scan_chunks = []
            for cid in probe:
                cl = clusters[cid]
                cl.access_count += 1
                self.tier.record_access(cid)
                if want_scan_ids:
                    if self.cfg.profiles_enabled and agent and cl.profiles.get(agent):
                        order = profile_order(cl.profiles[agent], cl.size)
                        scan_chunks.append(cl.member_ids[order])
                    else:
                        scan_chunks.append(cl.member_ids.copy())
            scan_ids = np.concatenate(scan_chunks) if scan_chunks else np.empty(0, dtype=np.int64)
            results.append(SearchResult(hits, stats, scan_ids))
        return results

    def _search_read_phase(self, agent, scopes, q, k, nprobe, internal, no_cache=False):
        """Store._search_read_phase (ref/engine.py:319-404) for one query:
        cache levels, staged items, coarse, probed lists with per-list early
        termination, _topk to max(k, kappa k).  Every distance comes out of
        ONE device pass (pk_agent_read): the FSM states (hint), the cache's
        pool rows and L1 centroids, the staged rows, the reference's coarse
        traversal and every row of the lists it probes (computed whether or
        not the cache stops first -- a few microseconds of device time against
        a round trip).  The hint, the scan orders and the stop rules then run
        over those values in the reference's order."""
        exhaustive_edge = k >= self.clusters.live_count()
        stats = SearchStats()
        use_cache = self.cfg.cache_enabled and agent and not no_cache
        cache = self.caches.get(agent) if use_cache else None
        table = self.patterns.get(agent) if (agent and self.cfg.pattern_enabled and not internal) else None
        lut, key = self.scope_codes.lut(scopes)
        rows = self.rows
        with rows.lock:
            parts = []
            plan = cache.read_plan(lut, key) if cache is not None else None
            if plan is not None:
                parts.append(plan["slots"])
            staged_parts = []
            for sc in sorted(scopes):  # staging areas: items not yet merged into clusters
                ss = self.clusters.staged_slots.get(sc)
                if ss:
                    ids = np.fromiter(ss.keys(), dtype=np.int64, count=len(ss))
                    sl = np.fromiter(ss.values(), dtype=np.int32, count=len(ss))
                    staged_parts.append(ids)
                    parts.append(sl)
            st_slots = table.state_slots() if table is not None else np.empty(0, np.int32)
            parts.append(st_slots)
            listing, lslots = [], None
            if table is not None and len(st_slots):
                lcache = self.caches.get(agent)
                if lcache is not None:
                    listing, lslots = lcache.l1_listing_slots()
            eff_nprobe, ef, mode = self._coarse_plan(k, nprobe)
            dev_nprobe = 0
            codes = None
            if self.clusters.clusters:
                in_scope = sum(len(self.clusters.by_scope[s]) for s in scopes)
                dev_nprobe = max(1, min(eff_nprobe, in_scope))
                codes = [self.scope_codes.intern(s) for s in sorted(scopes)]
                self.graph.upload()
            lists = self._prefetched_lists(q, (tuple(codes), dev_nprobe, ef, mode)) if dev_nprobe else None
            dall, SL, read_lists = self.index.agent_read(
                q, rows.take_puts(), np.concatenate(parts), st_slots if listing else None,
                lslots if listing else None, codes, 0 if lists is not None else dev_nprobe, ef, mode,
                cap=dev_nprobe * self._list_cap)
            if lists is None:
                lists = read_lists
        if lists is not None and len(lists[3]) > dev_nprobe * self._list_cap:
            self._list_cap = -(-len(lists[3]) // max(dev_nprobe, 1)) * 2
        n_plan = len(plan["slots"]) if plan is not None else 0
        at = n_plan
        staged_d = []
        for ids in staged_parts:
            staged_d.append(dall[at:at + len(ids)])
            at += len(ids)
        q_row = dall[at:at + len(st_slots)]
        hint = PatternHint()
        if table is not None:
            hint = self._hint_from(agent, q, q_row, listing, SL)
        id_chunks, dist_chunks, scan_chunks = [], [], []
        big = None
        early = False
        if cache is not None:
            cres = cache.replay(plan, dall[:n_plan], k, hint_keys=hint.predicted_clusters,
                                termination_enabled=not exhaustive_edge)
            if len(cres.ids):
                id_chunks.append(cres.ids)
                dist_chunks.append(cres.dists)
            scan_chunks.extend(cres.scan_ids)
            stats.scanned_vectors += cres.scanned
            early = cres.early_terminated
            stats.level_reached = cres.level_reached
            stats.early_terminated = early
        if not early:
            stats.level_reached = "L2"
            for ids, d in zip(staged_parts, staged_d):
                id_chunks.append(ids)
                dist_chunks.append(d)
                scan_chunks.append(ids)
                stats.scanned_vectors += len(ids)
            selected = []
            if lists is not None:
                cids, stats.coarse_computations, pre, all_ids, all_d = lists
                selected = [int(c) for c in cids if c >= 0]
            thresh = cache.threshold() if (cache is not None and not exhaustive_edge) else None
            clusters = self.clusters.clusters
            stop_at = len(selected)
            if thresh is not None and selected:
                # the stop rule after list li (k-th smallest of everything
                # scanned < thresh) holds exactly when >= k scanned distances
                # are below thresh: the first such li, from prefix counts
                below = sum(int(np.count_nonzero(c < thresh)) for c in dist_chunks)
                nsel = len(selected)
                # per-list counts by one segmented sum (a False sentinel keeps
                # every segment start in range; empty lists count 0)
                m2 = np.zeros(int(pre[nsel]) + 1, dtype=bool)
                np.less(all_d[:pre[nsel]], thresh, out=m2[:-1])
                cnt = np.add.reduceat(m2, pre[:nsel], dtype=np.int64)
                cnt[pre[:nsel] == pre[1:nsel + 1]] = 0
                cum = below + np.cumsum(cnt)
                ok = np.flatnonzero(cum >= k)
                if len(ok):
                    stop_at = int(ok[0]) + 1
                    early = True
                    stats.early_terminated = True
            for li in range(stop_at):
                cid = selected[li]
                cl = clusters[cid]
                cl.access_count += 1
                self.tier.record_access(cid)
                if self.cfg.profiles_enabled and agent and cl.profiles.get(agent):
                    order = profile_order(cl.profiles[agent], cl.size)
                    scan_chunks.append(cl.member_ids[order])
                else:
                    scan_chunks.append(cl.member_ids.copy())
            if stop_at:  # the scanned lists are one prefix of the device's rows
                n_rows = int(pre[stop_at])
                big = (all_ids[:n_rows], all_d[:n_rows])
                stats.scanned_vectors += n_rows
        extended = self._topk(id_chunks, dist_chunks, max(k, self.cfg.kappa * k), big)
        scan_ids = np.concatenate(scan_chunks) if scan_chunks else np.empty(0, dtype=np.int64)
        return SearchResult(extended[:k], stats, scan_ids), hint, extended

    # --- request sequences and their FSM distance rows ----------------------
    def _rows_for(self, agent, vecs):
        """D rows (distances to every pattern state, D's column layout) of
        request vectors, one device call."""
        table = self.patterns[agent]
        with self.rows.lock:
            st = table.state_slots()
            if not len(st) or not len(vecs):
                return [np.empty(0, np.float32) for _ in vecs]
            tmp = np.fromiter((self.rows.alloc(v) for v in vecs), dtype=np.int32, count=len(vecs))
            _, M, _ = self.index.agent_read(vecs[0], self.rows.take_puts(), np.empty(0, np.int32), tmp, st)
            self.rows.free_many(tmp)
        return [M[i].copy() for i in range(len(vecs))]

    def _seq_D(self, agent, last=None, last_row=None, window=None):
        """D = (request prefix [+ last]) x every pattern state: the cached
        rows, recomputed when missing or older than the patterns."""
        table = self.patterns[agent]
        seq = self.sequences[agent]
        drows = self._drows[agent]
        lo = 0 if window is None else max(0, len(seq) - window)
        need = [i for i in range(lo, len(seq)) if drows[i] is None or drows[i][0] != table.version]
        if need:
            fresh = self._rows_for(agent, [seq[i] for i in need])
            for i, r in zip(need, fresh):
                drows[i] = (table.version, r)
        rows_ = [drows[i][1] for i in range(lo, len(seq))]
        if last is not None:
            if last_row is None:
                last_row = self._rows_for(agent, [last])[0]
            rows_.append(last_row)
        if not rows_:
            return None
        return np.stack(rows_)

    def _hint_from(self, agent, q, q_row, listing, SL) -> PatternHint:
        """ref/engine.py:428-435 over the search's device values."""
        table = self.patterns[agent]
        w = self.cfg.request_window - 1
        prefix = self.sequences[agent][-w:] + [q] if w > 0 else [q]
        D = self._seq_D(agent, q, q_row, window=w) if table.fsms else None
        hint = table.match_and_predict(prefix, [(c, None) for c in listing], D,
                                       SL if listing else None)
        # the side effects key L0 by the same prefix's match: remember it
        self._match_memo[agent] = (q.tobytes(), len(self.sequences[agent]), hint.matched_fsm, q_row,
                                   table.version)
        self._qrow_memo[agent] = (q.tobytes(), len(self.sequences[agent]), q_row, table.version)
        return hint

    def _topk(self, id_chunks, dist_chunks, k, big=None):
        """ref/engine.py:406-426: lexsort by (dist, id), first occurrence per
        id, owners only (a cached copy of a deleted item is skipped).  Only a
        prefix of the order is ever consumed, so it sorts the smallest
        entries first (every entry tied with the cut is included) and falls
        back to the full order when duplicates / deleted ids exhaust it.
        ``big``: (ids, dists) of the probed lists' rows as one view, kept
        apart from the small chunks so they are not copied (the candidates
        of the cut come out of each part; the order over their union is the
        same whichever chunk an entry came from)."""
        if big is not None and len(big[0]) == 0:
            big = None
        if not id_chunks and big is None:
            return []
        ids = np.concatenate(id_chunks) if id_chunks else np.empty(0, np.int64)
        dists = np.concatenate(dist_chunks).astype(np.float32) if dist_chunks else np.empty(0, np.float32)
        if big is not None:
            bi, bd = big[0], big[1].astype(np.float32, copy=False)
        n = len(ids) + (len(bi) if big is not None else 0)
        take = min(n, 4 * k + 16)
        while True:
            if big is None:
                if take < n:
                    cut = np.partition(dists, take - 1)[take - 1]
                    sel = np.nonzero(dists <= cut)[0]  # ties at the cut kept whole
                else:
                    sel = np.arange(n)
                cids, cds = ids[sel], dists[sel]
            else:
                if take < n:
                    # the take-th smallest of the union: within the big part's
                    # take smallest and the small chunks
                    head = np.partition(bd, take - 1)[:take] if len(bd) > take else bd
                    cut = np.partition(np.concatenate((head, dists)), take - 1)[take - 1]
                    sb, ss = np.nonzero(bd <= cut)[0], np.nonzero(dists <= cut)[0]
                else:
                    sb, ss = np.arange(len(bd)), np.arange(len(dists))
                cids = np.concatenate((bi[sb], ids[ss]))
                cds = np.concatenate((bd[sb], dists[ss]))
            order = np.lexsort((cids, cds))
            hits, seen = [], set()
            owners, clusters = self.clusters.owner, self.clusters.clusters
            for iid, dv in zip(cids[order].tolist(), cds[order].tolist()):
                if iid in seen:
                    continue
                seen.add(iid)
                owner = owners.get(iid)
                if owner is None:
                    continue
                scope = owner[1] if owner[0] == "staged" else clusters[owner[1]].scope
                hits.append((iid, dv, scope))
                if len(hits) >= k:
                    return hits
            if len(cids) >= n:
                return hits
            take = min(n, 4 * take)

    def _state_key_for(self, agent, v, v_row=None):
        """ref/engine.py:437-446: the matched pattern's aligned state keys L0."""
        if not self.cfg.pattern_enabled:
            return DEFAULT_KEY
        table = self.patterns[agent]
        memo = self._match_memo.pop(agent, None)
        if memo is not None and memo[0] == v.tobytes() and memo[1] == len(self.sequences[agent]) \
                and memo[4] == table.version:
            idx, row = memo[2], memo[3]  # same prefix, same table: the hint's match
        else:
            prefix = self.sequences[agent][-(self.cfg.request_window - 1):] + [v]
            D = self._seq_D(agent, v, v_row, window=self.cfg.request_window - 1) if table.fsms else None
            idx, _ = table.match(prefix, D)
            row = None if D is None else D[-1]
        if idx is None:
            return DEFAULT_KEY
        if row is None:
            return (idx, table.fsms[idx].align(v, self.metric))
        off = table._offsets()[idx]
        return (idx, int(np.argmin(row[off:off + len(table.fsms[idx].states)])))

    def _cache_items(self, hits, positions: bool = False):
        """(id, vector, scope code, staged=False) of the hits that are still
        live; with positions, (index in hits, item) pairs.  The vectors are
        views: the pools copy what they keep."""
        out = []
        code = self.scope_codes.code
        for pos, (iid, _, sc) in enumerate(hits):
            vec = self._vector_view(iid)
            if vec is not None:
                c = code.get(sc)
                item = (iid, vec, c if c is not None else self.scope_codes.intern(sc), False)
                out.append((pos, item) if positions else item)
        return out

    def _search_side_effects(self, agent, q, k, hint, result, extended, internal):
        """ref/engine.py:448-501."""
        cache = self.caches.get(agent) if self.cfg.cache_enabled else None
        if cache is not None and result.hits:
            if extended is None:  # bare pass: the extended list is the kappa k prefix
                extended = result.hits
            if not result.stats.early_terminated:
                if not internal:
                    cache.record_completed(float(np.mean([h[1] for h in result.hits])))
            elif cache.verify_mode and not internal:
                self.runner.submit("search", self._verify_early_return, agent, q, k, result)
            state_key = self._state_key_for(agent, q)
            # the hits are the extended list's first k entries: one lookup each
            ext_items = self._cache_items(extended, positions=True)
            nh = len(result.hits)
            hit_items = [it for pos, it in ext_items if pos < nh] if extended[:nh] == result.hits \
                else [it for _, it in self._cache_items(result.hits, positions=True)]
            outcomes = cache.promote_and_capture(hit_items, state_key, q, [it for _, it in ext_items])
            if any(not o.empty for o in outcomes):
                with self._lock.write():
                    self._materialize(agent, outcomes)
        if self.cfg.profiles_enabled:
            by_cluster: dict[int, list[int]] = {}
            for iid, _, _ in result.hits:
                owner = self.clusters.owner.get(iid)
                if owner and owner[0] == "cluster":
                    cl = self.clusters.clusters[owner[1]]
                    by_cluster.setdefault(owner[1], []).append(cl.id_to_row[iid])
            for cid, rows in by_cluster.items():
                cl = self.clusters.clusters[cid]
                cl.profiles[agent] = profile_promote(cl.profiles.get(agent, []), rows,
                                                     self.cfg.p_size)
        if not internal:
            memo_row = None
            m = self._qrow_memo.pop(agent, None)
            if m is not None and m[0] == q.tobytes() and m[1] == len(self.sequences[agent]) \
                    and m[3] == self.patterns[agent].version:
                memo_row = m[2]
            self._append_sequence(agent, q, memo_row)
            if self.cfg.prefetch_enabled and not hint.empty:
                self.prefetch(agent, hint, k)

    def _verify_early_return(self, agent, q, k, early):
        """ref/engine.py:503-512: background full search vs an early return."""
        cache = self.caches[agent]
        full = self.search(agent, list(self.clusters.by_scope), q, k,
                           nprobe=max(len(self.clusters.clusters), 1), _internal=True, _no_cache=True)
        cache.verified_count += 1
        if early.ids != full.ids:
            cache.miss_count += 1
        if full.hits:
            cache.record_completed(float(np.mean([h[1] for h in full.hits])))

    def prefetch(self, agent, hint, k: int = 5):
        """ref/engine.py:524-555: repopulate the predicted L0 entry."""
        if hint.empty or hint.predicted_state is None:
            return
        key = hint.predicted_clusters[0] if hint.predicted_clusters else None
        cache = self.caches.get(agent)
        if cache is None or key is None or key in cache.l0:
            return
        token = (agent, key)
        if token in self._prefetch_inflight:
            return
        self._prefetch_inflight.add(token)

        def run():
            try:
                res = self.search(agent, list(self.clusters.by_scope), hint.predicted_state.c, k,
                                  _internal=True)
                if res.hits and cache is not None:
                    self._materialize(agent, cache.promote_to_l0(self._cache_items(res.hits), key))
            finally:
                self._prefetch_inflight.discard(token)

        self.runner.submit("cache", run)

    def _materialize(self, agent, outcomes):
        """ref/engine.py:662-678: merged-down staged items become base clusters.
        Returns the ids that were merged."""
        merged_all = set()
        for outcome in outcomes:
            for scope_code, items in outcome.staged.items():
                scope = self.scope_codes.name[scope_code]
                live = [(iid, vec) for iid, vec in items
                        if self.clusters.owner.get(iid) == ("staged", scope)]
                if not live:
                    continue
                self.clusters.create_cluster(scope, live)
                self.clusters.consume_staged(scope, [iid for iid, _ in live])
                merged = {iid for iid, _ in live}
                for c in self.caches.values():
                    c.mark_merged(merged)
                merged_all |= merged
        return merged_all

    # --- mutation ---------------------------------------------------------
    def insert(self, agent, scope: str, vectors, payloads=None, ids=None) -> list[int]:
        """ref/engine.py:557-569."""
        with self._serialized(agent):
            with self._lock.write():
                accepted = self._insert_impl(agent, scope, vectors, payloads, ids)
                self._tick(locked=True)
            return accepted

    def _insert_impl(self, agent, scope, vectors, payloads=None, ids=None) -> list[int]:
        """ref/engine.py:571-605 on the direct-place path, with the batch's
        assignments computed in one device call and recomputed only after a
        centroid change."""
        self._check_writable(agent, scope)
        vecs = self._vectors(vectors)
        if payloads is None:
            payloads = [b""] * len(vecs)
        if len(payloads) != len(vecs):
            raise UsageError("vectors and payloads must have equal length")
        if ids is not None:
            if len(ids) != len(vecs):
                raise UsageError("vectors and ids must have equal length")
            for iid in ids:
                if iid in self.clusters.owner:
                    raise UsageError(f"item id {iid} already live")
        accepted: list[int] = []
        n = len(vecs)
        i = 0
        assigned = None
        assigned_from = -1
        cache = self.caches.get(agent) if (self.cfg.cache_enabled and agent) else None
        # the vectors' FSM distance rows (state keys, request prefix): one call
        vrows = [None] * n
        if agent is not None and self.cfg.pattern_enabled and self.patterns[agent].fsms:
            vrows = self._rows_for(agent, vecs)
        if cache is not None:  # staged, owned by the agent's cache until merge-down
            # every vector's L0 promotion in order, their L1 side in one
            # placement chain (MultiLevelCache.promote_many_to_l0)
            code = self.scope_codes.intern(scope)
            proms = []
            for i in range(n):
                vec = vecs[i]
                iid = self._take_id(ids[i] if ids is not None else None)
                payload = payloads[i]
                self.payloads[iid] = payload.encode("utf-8") if isinstance(payload, str) else payload
                state_key = self._state_key_for(agent, vec, vrows[i])
                self.clusters.stage_item(scope, iid, vec)
                proms.append(([(iid, vec, code, True)], state_key))
                self._append_sequence(agent, vec, vrows[i])
                accepted.append(iid)
            cache.promote_many_to_l0(proms, lambda outs: self._materialize(agent, outs))
            return accepted
        while i < n:
            vec = vecs[i]
            iid = self._take_id(ids[i] if ids is not None else None)
            payload = payloads[i]
            if isinstance(payload, str):
                payload = payload.encode("utf-8")
            self.payloads[iid] = payload
            cands = self.clusters.by_scope[scope]
            if not cands:
                self.clusters.create_cluster(scope, [(iid, vec)])
                assigned = None
                if agent is not None:
                    self._append_sequence(agent, vec, vrows[i])
                accepted.append(iid)
                i += 1
                continue
            if assigned is None:
                assigned = self.clusters.assign_nearest_batch(vecs[i:], scope)
                assigned_from = i
            # the longest run of vectors whose inserts fire no split and no
            # maintenance (the reference checks after every vector,
            # ref/engine.py:647-660): placed together, in order, then the
            # firing vector's cluster mutates and later vectors re-assign
            j, fired = self._insert_run(assigned, assigned_from, i, n)
            run_ids = [iid] + [self._take_id(ids[t] if ids is not None else None)
                               for t in range(i + 1, j)]
            for t in range(i + 1, j):
                p_ = payloads[t]
                self.payloads[run_ids[t - i]] = p_.encode("utf-8") if isinstance(p_, str) else p_
            run_cids = assigned[i - assigned_from:j - assigned_from]
            self.tier.buffered_insert_batch(run_cids, np.asarray(run_ids, dtype=np.int64), vecs[i:j])
            if fired:
                self._after_cluster_mutation(int(run_cids[-1]))
                assigned = None  # a centroid moved: later vectors re-assign
            if agent is not None:
                for t in range(i, j):
                    self._append_sequence(agent, vecs[t], vrows[t])
            accepted.extend(run_ids)
            i = j
        return accepted

    def _vectors(self, vectors) -> np.ndarray:
        """The batch as one [n, d] float32 matrix with as_vector's checks
        (ref/core.py:74-86): validated in one pass; anything irregular goes
        through as_vector row by row for the same error."""
        d = self.cfg.dimension
        try:
            m = np.ascontiguousarray(vectors, dtype=np.float32)
        except (ValueError, TypeError):
            m = None
        if m is None or m.ndim != 2 or m.shape[1] != d or not np.isfinite(m).all():
            rows = [as_vector(v, d) for v in vectors]  # raises the reference's error
            return np.stack(rows) if rows else np.empty((0, d), np.float32)
        return m

    def _insert_run(self, assigned, base: int, i: int, n: int):
        """(j, fired): vectors i..j-1 go to their assigned clusters; fired when
        the insert of vector j-1 makes its cluster split or recompute (the
        predicates _after_cluster_mutation evaluates after each insert)."""
        clusters = self.clusters.clusters
        split_at = self.clusters.split_threshold if self.cfg.splits_enabled else None
        maint_at = self.clusters.maintenance_interval if self.cfg.lazy_maintenance else None
        added: dict[int, int] = {}
        j = i
        while j < n:
            cid = int(assigned[j - base])
            k = added.get(cid, 0) + 1
            added[cid] = k
            cl = clusters[cid]
            j += 1
            if (split_at is not None and cl.size + k >= split_at) or \
                    (maint_at is not None and cl.dirty + k >= maint_at):
                return j, True
        return j, False

    def _take_id(self, explicit) -> int:
        if explicit is None:
            iid = self._next_item_id
            self._next_item_id += 1
            return iid
        self._next_item_id = max(self._next_item_id, explicit + 1)
        return explicit

    def _after_cluster_mutation(self, cid: int) -> bool:
        """ref/engine.py:656-660; True when a centroid changed."""
        if self.cfg.splits_enabled and self.clusters.needs_split(cid):
            self.tier.split_offload(cid)
            return True
        if self.cfg.lazy_maintenance:
            cl = self.clusters.clusters.get(cid)
            if cl is not None and cl.dirty >= self.clusters.maintenance_interval:
                self.clusters.maintenance(cid)
                return True
        return False

    def bulk_build(self, scope: str, vectors, payloads=None) -> list[int]:
        """ref/engine.py:615-645 (k-means on device)."""
        with self._serialized(None), self._lock.write():
            self._check_writable(None, scope)
            mat = as_matrix(vectors, self.cfg.dimension) if len(vectors) else np.empty(
                (0, self.cfg.dimension), np.float32)
            n = len(mat)
            if n == 0:
                return []
            ids = [self._take_id(None) for _ in range(n)]
            if payloads is not None:
                for iid, p in zip(ids, payloads):
                    self.payloads[iid] = p.encode("utf-8") if isinstance(p, str) else p
            k = max(1, -(-n // self.cfg.split_target))
            id_arr = np.asarray(ids, dtype=np.int64)
            if k == 1:
                self.clusters.create_cluster(scope, (id_arr, mat))
                return ids
            center = vector_mean(mat)
            spread = vector_spread(mat, center, Metric.SQUARED_EUCLIDEAN)
            labels, _ = kmeans_split_points(mat, k, self.rng, spread, device=self.cfg.device)
            order = np.argsort(labels, kind="stable")  # each cluster's rows in row order
            bounds = np.concatenate([[0], np.cumsum(np.bincount(labels))])
            for c in range(int(labels.max()) + 1):
                rows = order[bounds[c]:bounds[c + 1]]
                if len(rows):
                    self.clusters.create_cluster(scope, (id_arr[rows], mat[rows]))
            return ids

    def update(self, agent, item_id: int, vector=None, payload=None) -> bool:
        """ref/engine.py:680-694."""
        with self._serialized(agent), self._lock.write():
            owner = self.clusters.owner.get(item_id)
            if owner is None:
                return False
            scope = owner[1] if owner[0] == "staged" else self.clusters.clusters[owner[1]].scope
            self._check_writable(agent, scope)
            old_vec = self._vector_of(item_id)
            new_vec = as_vector(vector, self.cfg.dimension) if vector is not None else old_vec
            new_payload = payload if payload is not None else self.payloads.get(item_id, b"")
            self._delete_internal(item_id)
            self._insert_impl(agent, scope, [new_vec], [new_payload], ids=[item_id])
            self._tick(locked=True)
            return True

    def delete(self, agent, item_id: int) -> bool:
        """ref/engine.py:696-705."""
        with self._serialized(agent), self._lock.write():
            owner = self.clusters.owner.get(item_id)
            if owner is None:
                return False
            scope = owner[1] if owner[0] == "staged" else self.clusters.clusters[owner[1]].scope
            self._check_writable(agent, scope)
            ok = self._delete_internal(item_id)
            self._tick(locked=True)
            return ok

    def _delete_internal(self, item_id: int) -> bool:
        owner = self.clusters.owner.get(item_id)
        if owner is None:
            return False
        if owner[0] == "cluster":
            cid = owner[1]
            self.clusters.delete_item(item_id)
            if cid in self.clusters.clusters and self.cfg.lazy_maintenance:
                self.clusters.maintenance(cid)
        else:
            self.clusters.delete_item(item_id)
        for c in self.caches.values():
            c.drop_item(item_id)
        self.payloads.pop(item_id, None)
        return True

    def end_request(self, agent: str):
        """ref/engine.py:724-731: fold the finished request into the agent's patterns."""
        if agent not in self.sequences:
            raise UsageError(f"unknown agent {agent!r}")
        seq = self.sequences[agent]
        if seq and self.cfg.pattern_enabled:
            table = self.patterns[agent]
            D = self._seq_D(agent) if table.fsms else None
            table.observe_completed(seq, D)
        self.sequences[agent] = []
        self._drows[agent] = []

    def _append_sequence(self, agent: str, v: np.ndarray, row=None):
        seq = self.sequences[agent]
        drows = self._drows[agent]
        seq.append(v)
        drows.append(None if row is None else (self.patterns[agent].version, row))
        if len(seq) > self.cfg.request_window:
            del seq[0]
            del drows[0]

    def flush_caches(self):
        """ref/engine.py:739-743: merge every cache level down."""
        with self._lock.write():
            for agent, cache in self.caches.items():
                self._materialize(agent, cache.flush())

    def _tick(self, locked: bool = False):
        """ref/engine.py:745-752: the hotset policy runs every hotset_interval
        operations (only the native cold tier has a budget to enforce)."""
        self._op_count += 1
        if self.tier.native and self._op_count % self.cfg.hotset_interval == 0:
            if locked:
                self.tier.hotset_update()
            else:
                with self._lock.write():
                    self.tier.hotset_update()

    # --- item access -------------------------------------------------------
    def _vector_of(self, item_id: int):
        v = self._vector_view(item_id)
        return None if v is None else v.copy()

    def _vector_view(self, item_id: int):
        owner = self.clusters.owner.get(item_id)
        if owner is None:
            return None
        if owner[0] == "staged":
            return self.clusters.staged[owner[1]].get(item_id)
        cl = self.clusters.clusters[owner[1]]
        row = cl.id_to_row.get(item_id)
        return cl.vectors[row] if row is not None else None

    def get_item(self, item_id: int):
        vec = self._vector_of(item_id)
        if vec is None:
            return None
        owner = self.clusters.owner[item_id]
        scope = owner[1] if owner[0] == "staged" else self.clusters.clusters[owner[1]].scope
        return vec, self.payloads.get(item_id, b""), scope

    def live_count(self) -> int:
        return self.clusters.live_count()

    def split_cluster(self, cid: int) -> SplitOutcome:
        return self.tier.split_offload(cid)

    # --- async surface ------------------------------------------------------
    def submit_batch(self, batch: OperationBatch):
        """ref/engine.py:784-801.  A homogeneous search batch (same scopes, k,
        nprobe) runs as one device pass."""

        def run():
            if batch.kind == "search" and batch.ops:
                groups = {}
                for op in batch.ops:
                    scopes, _q, k, *rest = op
                    key = (tuple(sorted(scopes)), k, rest[0] if rest else None)
                    groups.setdefault(key, 0)
                if len(groups) == 1:
                    scopes, _, k, *rest = batch.ops[0]
                    Q = np.stack([np.asarray(op[1], dtype=np.float32) for op in batch.ops])
                    return self.search_batch(batch.agent, scopes, Q, k, rest[0] if rest else None,
                                             want_scan_ids=True)
            out = []
            for op in batch.ops:
                if batch.kind == "search":
                    out.append(self.search(batch.agent, *op))
                elif batch.kind == "insert":
                    out.append(self.insert(batch.agent, *op))
                elif batch.kind == "update":
                    out.append(self.update(batch.agent, *op))
                else:
                    out.append(self.delete(batch.agent, *op))
            return out

        role = "search" if batch.kind == "search" else "update"
        return self.runner.submit(role, run)

    def submit_search(self, agent, scopes, q, k, nprobe=None):
        return self.runner.submit("search", self.search, agent, scopes, q, k, nprobe)

    def submit_insert(self, agent, scope, vectors, payloads=None):
        return self.runner.submit("update", self.insert, agent, scope, vectors, payloads)

    # --- persistence / ingestion -------------------------------------------
    def snapshot(self, path):
        """ref/engine.py:811-812 -> ref/persist.py:136-241 (same file format)."""
        from . import persist

        self.index.flush()
        persist.snapshot(self, path)

    @classmethod
    def restore(cls, path, **overrides) -> "Store":
        """ref/engine.py:814-816 -> ref/persist.py:244-380; ``overrides`` sets
        this package's own StoreConfig fields (``device``, ``sharded``)."""
        from . import persist

        return persist.restore(cls, path, **overrides)

    def export_ivf(self, path, scopes=None):
        """ref/persist.py:386-394."""
        if scopes is None:
            scopes = list(self.clusters.by_scope)
        cids = sorted(c for c, cl in self.clusters.clusters.items() if cl.scope in scopes)
        pnck.write_pnck(path, self.cfg.dimension, self.metric,
                        [(self.clusters.clusters[c].centroid, self.clusters.clusters[c].member_ids,
                          self.clusters.clusters[c].vectors) for c in cids])

    def load_external_ivf(self, path, scope: str) -> int:
        """ref/persist.py:397-424: import PNCK records as clusters of `scope`
        (centroids recomputed from the members, on device)."""
        if scope not in self.clusters.by_scope:
            raise UsageError(f"unknown scope {scope!r}")
        dimension, metric, records = pnck.read_pnck(path)
        if dimension != self.cfg.dimension:
            raise UsageError(
                f"dimension mismatch: file has {dimension}, store has {self.cfg.dimension}")
        if metric is not self.metric:
            raise UsageError(f"metric mismatch: file has {metric}, store has {self.metric}")
        return self.load_lists(scope, [(ids, rows) for _, ids, rows in records])

    def load_lists(self, scope: str, lists) -> int:
        """Import ready-made posting lists [(ids, rows)] into `scope`."""
        with self._serialized(None), self._lock.write():
            for ids, _ in lists:
                for iid in np.asarray(ids).tolist():
                    if iid in self.clusters.owner:
                        raise UsageError(f"item id {iid} already live in store")
            count = 0
            for ids, rows in lists:
                ids = np.asarray(ids, dtype=np.int64)
                if len(ids) == 0:
                    continue
                self.clusters.create_cluster(scope, (ids, rows))
                self._next_item_id = max(self._next_item_id, int(ids.max()) + 1)
                count += 1
            return count

    def ingest_fvecs(self, path, scope: str, limit: int | None = None) -> list[int]:
        import struct

        from .core import ParseError

        vecs = []
        with open(path, "rb") as f:
            offset = 0
            while True:
                head = f.read(4)
                if not head:
                    break
                if len(head) != 4:
                    raise ParseError("truncated fvecs record header", offset)
                d = struct.unpack("<i", head)[0]
                if d <= 0:
                    raise ParseError(f"bad fvecs dimension {d}", offset)
                if d != self.cfg.dimension:
                    raise UsageError(f"dimension mismatch: fvecs has {d}, expected {self.cfg.dimension}")
                body = f.read(4 * d)
                if len(body) != 4 * d:
                    raise ParseError("truncated fvecs record body", offset + 4)
                vecs.append(np.frombuffer(body, dtype=np.float32).copy())
                offset += 4 + 4 * d
                if limit is not None and len(vecs) >= limit:
                    break
        return self.insert(None, scope, vecs)

    def ingest_jsonl(self, path) -> int:
        """ref/engine.py:828-839 over ref/persist.py:464-477's records
        ({id?, vector, payload?, scope} per line), one insert each."""
        import json

        from .core import ParseError

        count = 0
        with open(path, "r", encoding="utf-8") as f:
            for lineno, line in enumerate(f, 1):
                line = line.strip()
                if not line:
                    continue
                try:
                    rec = json.loads(line)
                except json.JSONDecodeError as e:
                    raise ParseError(f"bad JSON on line {lineno}: {e.msg}", e.pos) from e
                if "vector" not in rec or "scope" not in rec:
                    raise ParseError(f"line {lineno} missing vector/scope", 0)
                self.insert(None, rec["scope"], [rec["vector"]], [rec.get("payload", "")],
                            ids=[rec["id"]] if "id" in rec else None)
                count += 1
        return count
