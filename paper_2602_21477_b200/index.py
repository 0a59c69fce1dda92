"""DeviceIndex: Python handle on one device-resident IVF (the C-ABI pk_index).

Owns the HBM arena of posting lists, the list table and the centroid table
of one GPU.  It is the storage half of the reference's ``ClusterStore``
(ref/clusters.py:186-362) plus the residency half of ``TierManager``
(ref/tiering.py:175-448): every list the store owns is resident here.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native as N


def _is_device_tensor(a) -> bool:
    return hasattr(a, "is_cuda") and a.is_cuda


def block_bytes(B: int, kk: int) -> int:
    from .sharded import block_offsets

    return block_offsets(B, kk)["total"]


class SearchOutput:
    """Batched search result arrays (host)."""

    __slots__ = ("ids", "dists", "cids", "counts", "probe", "scanned")

    def __init__(self, ids, dists, cids, counts, probe, scanned):
        self.ids = ids
        self.dists = dists
        self.cids = cids
        self.counts = counts
        self.probe = probe
        self.scanned = scanned


class DeviceIndex:
    def __init__(self, dimension: int, metric_code: int = 0, device: int = 0,
                 reserve_rows: int = 0, reserve_lists: int = 0):
        self.dimension = int(dimension)
        self.metric_code = int(metric_code)
        self.device = int(device)
        h = ctypes.c_void_p()
        N.check(N.lib().pk_index_create(self.dimension, self.metric_code, self.device,
                                        int(reserve_rows), int(reserve_lists), ctypes.byref(h)))
        self._h = h
        self._pend: list = []  # queued appends (flushed before any other operation)
        self._pend_lock = threading.Lock()
        self._next_slot = 0

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h is not None and self._h.value:
            self.flush()
            N.lib().pk_index_destroy(self._h)
        self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        self.flush()
        N.check(N.lib().pk_sync(self._h))

    def nbytes(self) -> int:
        self.flush()
        v = ctypes.c_int64(0)
        N.check(N.lib().pk_index_bytes(self._h, ctypes.byref(v)))
        return int(v.value)

    # ---- posting lists -------------------------------------------------
    def create_list(self, cid: int, scope_code: int, rows, ids) -> np.ndarray:
        self.flush()
        if _is_device_tensor(rows):
            return self.create_list_device(cid, scope_code, rows, ids)
        rows = N.f32(rows, self.dimension)
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        cent = np.empty(self.dimension, dtype=np.float32)
        N.check(N.lib().pk_list_create(self._h, int(cid), int(scope_code), N.ptr(rows), N.ptr(ids),
                                       len(ids), N.ptr(cent), 0))
        return cent

    def create_list_device(self, cid: int, scope_code: int, rows, ids) -> np.ndarray:
        """rows/ids are device tensors ([n, d] f32 contiguous, [n] i64)."""
        self.flush()
        cent = np.empty(self.dimension, dtype=np.float32)
        N.check(N.lib().pk_list_create(self._h, int(cid), int(scope_code), N.ptr(rows), N.ptr(ids),
                                       int(ids.shape[0]), N.ptr(cent), N.PK_DEVICE_PTRS))
        return cent

    def stream_handle(self) -> int:
        return int(N.lib().pk_stream(self._h) or 0)

    def profile_begin(self):
        N.check(N.lib().pk_profile_begin(self._h))

    def profile_end(self):
        out = np.zeros(len(N.STAGES), dtype=np.float64)
        calls = ctypes.c_int32(0)
        N.check(N.lib().pk_profile_end(self._h, N.ptr(out), len(out), ctypes.byref(calls)))
        return dict(zip(N.STAGES, out.tolist())), int(calls.value)

    def pool_counts(self, B: int) -> np.ndarray:
        """Candidate-pool size per query of the last screened search."""
        out = np.empty(B, dtype=np.int32)
        N.check(N.lib().pk_debug_pool_counts(self._h, N.ptr(out), B))
        return out

    def coarse_counts(self, B: int) -> np.ndarray:
        """Lists re-ranked exactly per query by the last tensor-core coarse pass."""
        out = np.empty(B, dtype=np.int32)
        N.check(N.lib().pk_debug_coarse_counts(self._h, N.ptr(out), B))
        return out

    def rerank_counts(self, B: int) -> np.ndarray:
        """Pool entries re-ranked exactly per query by the last screened search."""
        out = np.empty(B, dtype=np.int32)
        N.check(N.lib().pk_debug_rerank_counts(self._h, N.ptr(out), B))
        return out

    def append(self, cid: int, rows, ids):
        """Cluster.add (ref/clusters.py:71-79).  Appends are queued and sent as
        one pk_list_append_batch call (one H2D copy, one scatter kernel)
        before the next operation that reads the index; a usage error (e.g.
        a remote list) surfaces at that flush and leaves the index unchanged."""
        rows = N.f32(rows, self.dimension)
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        if len(ids):
            with self._pend_lock:
                self._pend.append((int(cid), rows, ids))

    def append_rows(self, cids, rows, ids):
        """Appends of several clusters at once (cids per row; each cluster's
        rows in order), queued like ``append``."""
        rows = N.f32(rows, self.dimension)
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        cids = np.ascontiguousarray(cids, dtype=np.int64)
        if len(ids):
            with self._pend_lock:
                self._pend.append((cids, rows, ids))

    def flush(self):
        if not self._pend:
            return
        with self._pend_lock:
            pend, self._pend = self._pend, []
        if not pend:
            return
        if len(pend) == 1 and isinstance(pend[0][0], np.ndarray):  # one append_rows (an insert run)
            cids, rows, ids = pend[0]
        else:
            cids = np.concatenate([c if isinstance(c, np.ndarray) else np.full(len(i), c, dtype=np.int64)
                                   for c, _, i in pend])
            rows = np.ascontiguousarray(np.concatenate([r for _, r, _ in pend]))
            ids = np.ascontiguousarray(np.concatenate([i for _, _, i in pend]))
        N.check(N.lib().pk_list_append_batch(self._h, len(ids), N.ptr(cids), N.ptr(rows), N.ptr(ids)))

    def remove_row(self, cid: int, row: int):
        self.flush()
        N.check(N.lib().pk_list_remove_row(self._h, int(cid), int(row)))

    def retire(self, cid: int):
        self.flush()
        N.check(N.lib().pk_list_retire(self._h, int(cid)))

    def recompute(self, cid: int) -> np.ndarray:
        self.flush()
        cent = np.empty(self.dimension, dtype=np.float32)
        N.check(N.lib().pk_list_recompute(self._h, int(cid), N.ptr(cent)))
        return cent

    def set_centroid(self, cid: int, centroid):
        self.flush()
        c = N.f32(centroid).reshape(-1)
        N.check(N.lib().pk_list_set_centroid(self._h, int(cid), N.ptr(c)))

    def size(self, cid: int) -> int:
        self.flush()
        v = ctypes.c_int64(0)
        N.check(N.lib().pk_list_size(self._h, int(cid), ctypes.byref(v)))
        return int(v.value)

    def read(self, cid: int):
        self.flush()
        n = self.size(cid)
        rows = np.empty((n, self.dimension), dtype=np.float32)
        ids = np.empty(n, dtype=np.int64)
        N.check(N.lib().pk_list_read(self._h, int(cid), N.ptr(rows), N.ptr(ids)))
        return rows, ids

    # ---- hot path ------------------------------------------------------
    def search(self, Q, scope_codes, nprobe: int, kk: int, want_probe: bool = False,
               want_scanned: bool = True) -> SearchOutput:
        self.flush()
        Q = N.f32(Q, self.dimension)
        B = Q.shape[0]
        codes = np.ascontiguousarray(scope_codes, dtype=np.int32)
        ids = np.empty((B, kk), dtype=np.int64)
        dd = np.empty((B, kk), dtype=np.float32)
        cids = np.empty((B, kk), dtype=np.int64)
        cnt = np.empty(B, dtype=np.int32)
        probe = np.empty((B, nprobe), dtype=np.int64) if want_probe else None
        scanned = np.empty(B, dtype=np.int64) if want_scanned else None
        N.check(N.lib().pk_search(self._h, N.ptr(Q), B, N.ptr(codes), len(codes), int(nprobe),
                                  int(kk), N.ptr(ids), N.ptr(dd), N.ptr(cids), N.ptr(cnt),
                                  N.ptr(probe), N.ptr(scanned), 0))
        return SearchOutput(ids, dd, cids, cnt, probe, scanned)

    def search_submit(self, Q, scope_codes, nprobe: int, kk: int):
        """Asynchronous search of a host batch (up to N.PK_ASYNC_SLOTS in
        flight, slots used round-robin: collect a ticket before submitting
        that many more); returns a ticket for search_collect.  Keep Q alive
        (ideally pinned) until collected."""
        self.flush()
        Q = N.f32(Q, self.dimension)
        slot = self._next_slot
        self._next_slot = (slot + 1) % N.PK_ASYNC_SLOTS
        codes = np.ascontiguousarray(scope_codes, dtype=np.int32)
        N.check(N.lib().pk_search_submit(self._h, slot, N.ptr(Q), Q.shape[0], N.ptr(codes), len(codes),
                                         int(nprobe), int(kk)))
        return (slot, Q.shape[0], int(kk), Q)

    def search_collect(self, ticket) -> SearchOutput:
        slot, B, kk, _ = ticket
        ids = np.empty((B, kk), dtype=np.int64)
        dd = np.empty((B, kk), dtype=np.float32)
        cids = np.empty((B, kk), dtype=np.int64)
        cnt = np.empty(B, dtype=np.int32)
        scanned = np.empty(B, dtype=np.int64)
        N.check(N.lib().pk_search_collect(self._h, slot, N.ptr(ids), N.ptr(dd), N.ptr(cids), N.ptr(cnt),
                                          N.ptr(scanned)))
        return SearchOutput(ids, dd, cids, cnt, None, scanned)

    def search_device(self, Q, scope_codes, nprobe: int, kk: int, out_ids, out_d, out_cid,
                      out_n, out_scanned=None):
        """Device-pointer variant (torch tensors on this device); async on the
        index stream."""
        self.flush()
        N.check(N.lib().pk_search(self._h, N.ptr(Q), Q.shape[0], N.ptr(scope_codes),
                                  scope_codes.shape[0], int(nprobe), int(kk), N.ptr(out_ids),
                                  N.ptr(out_d), N.ptr(out_cid), N.ptr(out_n), None,
                                  N.ptr(out_scanned), N.PK_DEVICE_PTRS))

    # ---- the reference's hybrid coarse graph (pk_graph_*) -----------------------
    def graph_set(self, M: int, node_cids, node_levels, nbr, por_ptr, por, static_code: int,
                  scope_codes, scope_entries, scope_maxl):
        self.flush()
        arr = lambda a, t: np.ascontiguousarray(a, dtype=t)  # noqa: E731
        nc, nl, nb = arr(node_cids, np.int64), arr(node_levels, np.int32), arr(nbr, np.int64)
        pp, pv = arr(por_ptr, np.int64), arr(por, np.int64)
        sc, se, sm = arr(scope_codes, np.int32), arr(scope_entries, np.int64), arr(scope_maxl, np.int32)
        N.check(N.lib().pk_graph_set(self._h, int(M), len(nc), N.ptr(nc), N.ptr(nl), N.ptr(nb), N.ptr(pp),
                                     N.ptr(pv), int(static_code), len(sc), N.ptr(sc), N.ptr(se), N.ptr(sm)))

    def search_graph(self, Q, scope_codes, nprobe: int, kk: int, ef: int, mode: int = 0,
                     want_probe: bool = False):
        """pk_search with the reference's graph traversal as the coarse stage;
        returns (SearchOutput, coarse distance computations i32[B])."""
        self.flush()
        Q = N.f32(Q, self.dimension)
        B = Q.shape[0]
        codes = np.ascontiguousarray(scope_codes, dtype=np.int32)
        ids = np.empty((B, kk), dtype=np.int64)
        dd = np.empty((B, kk), dtype=np.float32)
        cids = np.empty((B, kk), dtype=np.int64)
        cnt = np.empty(B, dtype=np.int32)
        probe = np.empty((B, nprobe), dtype=np.int64) if want_probe else None
        scanned = np.empty(B, dtype=np.int64)
        coarse = np.empty(B, dtype=np.int32)
        N.check(N.lib().pk_search_graph(self._h, N.ptr(Q), B, N.ptr(codes), len(codes), int(nprobe),
                                        int(ef), int(mode), int(kk), N.ptr(ids), N.ptr(dd), N.ptr(cids),
                                        N.ptr(cnt), N.ptr(probe), N.ptr(scanned), N.ptr(coarse), 0))
        return SearchOutput(ids, dd, cids, cnt, probe, scanned), coarse

    def search_graph_block(self, Q, scope_codes, nprobe: int, kk: int, ef: int, mode: int = 0):
        """search_graph written as one shard result block (host uint8) plus the
        probe cids and coarse counts (the sharded Store)."""
        from .sharded import block_views

        self.flush()
        Q = N.f32(Q, self.dimension)
        B = Q.shape[0]
        codes = np.ascontiguousarray(scope_codes, dtype=np.int32)
        blk = np.zeros(block_bytes(B, kk), dtype=np.uint8)
        ids, cids, scanned, dd, cnt = block_views(blk, B, kk)
        probe = np.empty((B, nprobe), dtype=np.int64)
        coarse = np.empty(B, dtype=np.int32)
        N.check(N.lib().pk_search_graph(self._h, N.ptr(Q), B, N.ptr(codes), len(codes), int(nprobe),
                                        int(ef), int(mode), int(kk), N.ptr(ids), N.ptr(dd), N.ptr(cids),
                                        N.ptr(cnt), N.ptr(probe), N.ptr(scanned), N.ptr(coarse), 0))
        return blk, probe, coarse

    def graph_probe(self, Q, scope_codes, nprobe: int, ef: int, mode: int = 0):
        """Graph coarse stage only: (probed cids i64[B, nprobe], counts i32[B])."""
        self.flush()
        Q = N.f32(Q, self.dimension)
        codes = np.ascontiguousarray(scope_codes, dtype=np.int32)
        out = np.empty((Q.shape[0], nprobe), dtype=np.int64)
        coarse = np.empty(Q.shape[0], dtype=np.int32)
        N.check(N.lib().pk_graph_probe(self._h, N.ptr(Q), Q.shape[0], N.ptr(codes), len(codes), int(nprobe),
                                       int(ef), int(mode), N.ptr(out), N.ptr(coarse)))
        return out, coarse

    def centroid_dists(self, V):
        """(out f32[n, nslots], slot cids i64[nslots]): reference distances of
        host rows to every slot's centroid."""
        self.flush()
        V = N.f32(V, self.dimension)
        ns = ctypes.c_int32(0)
        N.check(N.lib().pk_slot_count(self._h, ctypes.byref(ns)))
        out = np.empty((V.shape[0], ns.value), dtype=np.float32)
        cids = np.empty(ns.value, dtype=np.int64)
        N.check(N.lib().pk_centroid_dists(self._h, N.ptr(V), V.shape[0], N.ptr(out), N.ptr(cids)))
        return out, cids

    def list_slot(self, cid: int) -> int:
        v = ctypes.c_int32(0)
        N.check(N.lib().pk_list_slot(self._h, int(cid), ctypes.byref(v)))
        return int(v.value)

    # ---- agent-mode L2 scan ---------------------------------------------------
    def coarse_cids(self, Q, scope_codes, nprobe: int) -> np.ndarray:
        """Coarse stage only: probed list ids i64[B, nprobe] in coarse order."""
        self.flush()
        Q = N.f32(Q, self.dimension)
        codes = np.ascontiguousarray(scope_codes, dtype=np.int32)
        out = np.empty((Q.shape[0], nprobe), dtype=np.int64)
        N.check(N.lib().pk_search_coarse_cids(self._h, N.ptr(Q), Q.shape[0], N.ptr(codes), len(codes),
                                              int(nprobe), N.ptr(out)))
        return out

    def scan_lists(self, q, cids, total: int):
        """Distances of one query to every row of the lists ``cids`` in that
        order: (ids i64[total], dists f32[total], prefix i64[m + 1])."""
        self.flush()
        q = N.f32(q).reshape(-1)
        cids = np.ascontiguousarray(cids, dtype=np.int64)
        ids = np.empty(max(total, 1), dtype=np.int64)
        dd = np.empty(max(total, 1), dtype=np.float32)
        pre = np.zeros(len(cids) + 1, dtype=np.int64)
        N.check(N.lib().pk_scan_lists(self._h, N.ptr(q), N.ptr(cids), len(cids), N.ptr(ids), N.ptr(dd),
                                      N.ptr(pre)))
        return ids[:pre[-1]], dd[:pre[-1]], pre

    # ---- agent path: one device pass per agent search (pk_agent.cu) ---------
    def rows_reserve(self, n: int):
        """Capacity for n row-store slots (pk_rows_reserve)."""
        N.check(N.lib().pk_rows_reserve(self._h, int(n)))

    def rows_put(self, slots, rows):
        """Rows into the HBM row store at the given slots (pk_rows_put)."""
        self.flush()
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        rows = N.f32(rows, self.dimension)
        N.check(N.lib().pk_rows_put(self._h, N.ptr(slots), N.ptr(rows), len(slots)))

    def agent_read(self, q, puts, slots, mq=None, mx=None, scope_codes=None, nprobe: int = 0,
                   ef: int = 0, mode: int = 0, cap: int = 0):
        """pk_agent_read: (d f32[len(slots)], m f32[len(mq), len(mx)],
        lists) where lists = (cids i64[nprobe], coarse, prefix i64[nprobe+1],
        ids, dists) or None when nprobe == 0."""
        self.flush()
        q = N.f32(q).reshape(-1)
        ps, pr = puts if puts is not None else (None, None)
        nput = 0 if ps is None else len(ps)
        if nput:
            ps = np.ascontiguousarray(ps, dtype=np.int32)
            pr = N.f32(pr, self.dimension)
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        out_d = np.empty(max(len(slots), 1), dtype=np.float32)
        nmq = 0 if mq is None else len(mq)
        nmx = 0 if mx is None else len(mx)
        if nmq and nmx:
            mq = np.ascontiguousarray(mq, dtype=np.int32)
            mx = np.ascontiguousarray(mx, dtype=np.int32)
        else:
            nmq = nmx = 0
        out_m = np.empty((max(nmq, 1), max(nmx, 1)), dtype=np.float32)
        lists = None
        if nprobe > 0:
            codes = np.ascontiguousarray(scope_codes, dtype=np.int32)
            cids = np.empty(nprobe, dtype=np.int64)
            coarse = ctypes.c_int32(0)
            pre = np.zeros(nprobe + 1, dtype=np.int64)
            cap = max(int(cap), 1)
            while True:
                ids = np.empty(cap, dtype=np.int64)
                dd = np.empty(cap, dtype=np.float32)
                rc = N.lib().pk_agent_read(
                    self._h, N.ptr(q), N.ptr(ps) if nput else None, N.ptr(pr) if nput else None, nput,
                    N.ptr(slots), len(slots), N.ptr(out_d), N.ptr(mq) if nmq else None, nmq,
                    N.ptr(mx) if nmx else None, nmx, N.ptr(out_m), N.ptr(codes), len(codes), int(nprobe),
                    int(ef), int(mode), N.ptr(cids), ctypes.byref(coarse), N.ptr(pre), N.ptr(ids), N.ptr(dd),
                    cap)
                if rc != 0 and pre[-1] > cap:  # more rows than the guess: the puts are in; ask again
                    cap = int(pre[-1])
                    nput = 0
                    continue
                N.check(rc)
                break
            t = int(pre[-1])
            lists = (cids, int(coarse.value), pre, ids[:t], dd[:t])
        else:
            N.check(N.lib().pk_agent_read(
                self._h, N.ptr(q), N.ptr(ps) if nput else None, N.ptr(pr) if nput else None, nput,
                N.ptr(slots), len(slots), N.ptr(out_d), N.ptr(mq) if nmq else None, nmq,
                N.ptr(mx) if nmx else None, nmx, N.ptr(out_m), None, 0, 0, 0, 0, None, None, None, None,
                None, 0))
        return out_d[:len(slots)], out_m[:nmq, :nmx], lists

    def agent_lists(self, Q, scope_codes, nprobe: int, ef: int, mode: int, cap: int):
        """pk_agent_lists: the coarse traversal and probed-list rows of B
        queries in one pass.  Returns (version, [lists_b]) with lists_b as
        agent_read's lists, or None for a query whose rows exceed cap."""
        self.flush()
        Q = N.f32(Q, self.dimension)
        B = Q.shape[0]
        codes = np.ascontiguousarray(scope_codes, dtype=np.int32)
        cap = max(int(cap), 1)
        cids = np.empty((B, nprobe), dtype=np.int64)
        coarse = np.empty(B, dtype=np.int32)
        pre = np.zeros((B, nprobe + 1), dtype=np.int64)
        ids = np.empty((B, cap), dtype=np.int64)
        dd = np.empty((B, cap), dtype=np.float32)
        ver = ctypes.c_uint64(0)
        N.check(N.lib().pk_agent_lists(self._h, N.ptr(Q), B, N.ptr(codes), len(codes), int(nprobe), int(ef),
                                       int(mode), cap, N.ptr(cids), N.ptr(coarse), N.ptr(pre), N.ptr(ids),
                                       N.ptr(dd), ctypes.byref(ver)))
        out = []
        for b in range(B):
            t = int(pre[b, -1])
            out.append(None if t > cap else (cids[b], int(coarse[b]), pre[b], ids[b, :t], dd[b, :t]))
        return int(ver.value), out

    def list_version(self) -> int:
        """pk_list_version (after the queued appends are applied)."""
        self.flush()
        v = ctypes.c_uint64(0)
        N.check(N.lib().pk_list_version(self._h, ctypes.byref(v)))
        return int(v.value)

    def l1_place(self, nc, n_p, capacity, sums, cents, counts, items, item_ids, holder, q=None):
        """pk_l1_place: (targets i32[m], added u8[m], q target or None)."""
        self.flush()
        d = self.dimension
        m = len(items)
        sums = np.ascontiguousarray(sums, dtype=np.float64).reshape(nc, d)
        cents = N.f32(cents).reshape(nc, d)
        counts = np.ascontiguousarray(counts, dtype=np.int32)
        items = N.f32(items).reshape(m, d)
        holder = np.ascontiguousarray(holder, dtype=np.int32)
        item_ids = np.ascontiguousarray(item_ids, dtype=np.int64)
        qv = None if q is None else N.f32(q).reshape(d)
        tg = np.empty(max(m, 1), dtype=np.int32)
        added = np.empty(max(m, 1), dtype=np.uint8)
        merged = np.empty(max(m, 1), dtype=np.uint8)
        qt = ctypes.c_int32(-3)
        N.check(N.lib().pk_l1_place(self._h, int(nc), int(n_p), int(capacity), N.ptr(sums), N.ptr(cents),
                                    N.ptr(counts), N.ptr(items), N.ptr(item_ids), N.ptr(holder), m, N.ptr(qv),
                                    N.ptr(tg),
                                    N.ptr(added), N.ptr(merged), ctypes.byref(qt)))
        return tg[:m].tolist(), added[:m].tolist(), (int(qt.value) if q is not None else None)

    # ---- cold tier (TierManager residency, ref/tiering.py:175-448) --------
    TIER_STATS = ("resident_lists", "cold_lists", "resident_bytes", "staged_lists_last",
                  "staged_bytes_last", "staged_bytes_total", "staged_searches",
                  "admissions_started", "admissions_done", "host_arena_bytes",
                  "arena_top_rows", "arena_cap_rows")

    def enable_tier(self, reserve_rows: int = 0):
        """Cold tier on: lists live in pinned host memory, HBM holds the
        resident ones (call before creating lists)."""
        self.flush()
        N.check(N.lib().pk_index_enable_tier(self._h, int(reserve_rows)))

    def set_resident(self, cid: int, resident: bool):
        self.flush()
        N.check(N.lib().pk_list_set_resident(self._h, int(cid), 1 if resident else 0))

    def fail_next_alloc(self, n: int = 1):
        """Fault injection: the next n admissions fail (pk_debug_fail_next_alloc)."""
        N.check(N.lib().pk_debug_fail_next_alloc(self._h, int(n)))

    def residency(self, cid: int) -> int:
        """0 cold, 1 HBM-resident, 2 admission in flight."""
        self.flush()
        v = ctypes.c_int(0)
        N.check(N.lib().pk_list_residency(self._h, int(cid), ctypes.byref(v)))
        return int(v.value)

    def tier_stats(self) -> dict:
        self.flush()
        out = np.zeros(len(self.TIER_STATS), dtype=np.int64)
        N.check(N.lib().pk_tier_stats(self._h, N.ptr(out), len(out)))
        return dict(zip(self.TIER_STATS, out.tolist()))

    # ---- sharded search ---------------------------
    def add_remote_list(self, cid: int, scope_code: int, centroid):
        """A list owned by another rank: centroid only (joins the coarse
        quantizer, holds no rows here)."""
        self.flush()
        c = N.f32(centroid).reshape(-1)
        if c.shape[0] != self.dimension:
            raise N.UsageError("centroid dimension mismatch")
        N.check(N.lib().pk_list_add_remote(self._h, int(cid), int(scope_code), N.ptr(c)))

    def search_block(self, Q, scope_codes, nprobe: int, kk: int) -> np.ndarray:
        """Local search written as one shard result block (host uint8)."""
        self.flush()
        from .sharded import block_views

        Q = N.f32(Q, self.dimension)
        B = Q.shape[0]
        codes = np.ascontiguousarray(scope_codes, dtype=np.int32)
        blk = np.zeros(block_bytes(B, kk), dtype=np.uint8)
        ids, cids, scanned, dd, cnt = block_views(blk, B, kk)
        N.check(N.lib().pk_search(self._h, N.ptr(Q), B, N.ptr(codes), len(codes), int(nprobe),
                                  int(kk), N.ptr(ids), N.ptr(dd), N.ptr(cids), N.ptr(cnt), None,
                                  N.ptr(scanned), 0))
        return blk

    def search_block_device(self, Q, scope_codes, nprobe: int, kk: int, block):
        """Device variant: Q [B, d] f32 and block (uint8, block_bytes(B, kk))
        are tensors on this device; async on the index stream."""
        self.flush()
        from .sharded import block_offsets

        B = int(Q.shape[0])
        o = block_offsets(B, kk)
        base = block.data_ptr()
        N.check(N.lib().pk_search(self._h, N.ptr(Q), B, N.ptr(scope_codes), int(scope_codes.shape[0]),
                                  int(nprobe), int(kk), base + o["ids"], base + o["dists"],
                                  base + o["cids"], base + o["n"], None, base + o["scanned"],
                                  N.PK_DEVICE_PTRS))

    def centroid_of(self, rows) -> np.ndarray:
        """Cluster.recompute_stats centroid of host rows (the arithmetic
        create_list applies on the device)."""
        if _is_device_tensor(rows):
            out = np.empty(self.dimension, dtype=np.float32)
            dev_out = rows.new_empty(self.dimension)
            N.check(N.lib().pk_centroid(N.ptr(rows), int(rows.shape[0]), self.dimension,
                                        N.ptr(dev_out), N.PK_DEVICE_PTRS))
            out[:] = dev_out.cpu().numpy()
            return out
        from .kernels import centroid

        return centroid(N.f32(rows, self.dimension))

    def search_coarse(self, Q, scope_codes, nprobe: int) -> np.ndarray:
        """Coarse stage only: list handles int32[B, nprobe] (-1 padded)."""
        self.flush()
        Q = N.f32(Q, self.dimension)
        B = Q.shape[0]
        codes = np.ascontiguousarray(scope_codes, dtype=np.int32)
        out = np.empty((B, nprobe), dtype=np.int32)
        N.check(N.lib().pk_search_coarse(self._h, N.ptr(Q), B, N.ptr(codes), len(codes),
                                         int(nprobe), N.ptr(out), 0))
        return out

    def search_probed(self, Q, probe, kk: int, group: int) -> np.ndarray:
        """Scan stage only for given handles; B / group shard blocks (host)."""
        self.flush()
        Q = N.f32(Q, self.dimension)
        probe = np.ascontiguousarray(probe, dtype=np.int32)
        B, nprobe = probe.shape
        out = np.empty((B // group) * block_bytes(group, kk), dtype=np.uint8)
        N.check(N.lib().pk_search_probed(self._h, N.ptr(Q), B, N.ptr(probe), nprobe, int(kk),
                                         int(group), N.ptr(out), 0))
        return out

    def search_coarse_device(self, Q, scope_codes, nprobe: int, out_probe):
        self.flush()
        N.check(N.lib().pk_search_coarse(self._h, N.ptr(Q), int(Q.shape[0]), N.ptr(scope_codes),
                                         int(scope_codes.shape[0]), int(nprobe), N.ptr(out_probe),
                                         N.PK_DEVICE_PTRS))

    def search_probed_device(self, Q, probe, kk: int, group: int, out_blocks):
        self.flush()
        N.check(N.lib().pk_search_probed(self._h, N.ptr(Q), int(Q.shape[0]), N.ptr(probe),
                                         int(probe.shape[1]), int(kk), int(group),
                                         N.ptr(out_blocks), N.PK_DEVICE_PTRS))

    # ---- peer combine (pk_combine_*) -----------------------------------------
    def combine_create(self, R: int, my_rank: int, group: int, kk: int) -> bytes:
        """Receive area for the peer combine; returns its 64-byte IPC handle."""
        self.flush()
        h = ctypes.create_string_buffer(64)
        N.check(N.lib().pk_combine_create(self._h, int(R), int(my_rank), int(group), int(kk), h))
        return h.raw

    def combine_open(self, peer: int, handle: bytes | None = None, area_ptr: int | None = None):
        buf = ctypes.create_string_buffer(handle, 64) if handle is not None else None
        N.check(N.lib().pk_combine_open(self._h, int(peer), buf, area_ptr))

    def combine_area(self) -> int:
        return int(N.lib().pk_combine_area(self._h) or 0)

    def combine_search_probed_device(self, Q, probe, epoch: int):
        self.flush()
        N.check(N.lib().pk_combine_search_probed(self._h, N.ptr(Q), int(Q.shape[0]), N.ptr(probe),
                                                 int(probe.shape[1]), int(epoch), N.PK_DEVICE_PTRS))

    def combine_merge_device(self, epoch: int, out_ids, out_d, out_cid, out_n, out_scanned=None,
                             timeout_s: float = 10.0):
        N.check(N.lib().pk_combine_merge(self._h, int(epoch), float(timeout_s), N.ptr(out_ids),
                                         N.ptr(out_d), N.ptr(out_cid), N.ptr(out_n), N.ptr(out_scanned),
                                         N.PK_DEVICE_PTRS))

    def combine_status(self) -> int:
        v = ctypes.c_int32(0)
        N.check(N.lib().pk_combine_status(self._h, ctypes.byref(v)))
        return int(v.value)

    def merge_shards(self, blocks, R: int, B: int, kk: int):
        """Host: blocks uint8[R * block_bytes] -> (ids, dists, cids, counts, scanned)."""
        blocks = np.ascontiguousarray(blocks, dtype=np.uint8)
        ids = np.empty((B, kk), dtype=np.int64)
        dd = np.empty((B, kk), dtype=np.float32)
        cids = np.empty((B, kk), dtype=np.int64)
        cnt = np.empty(B, dtype=np.int32)
        sc = np.empty(B, dtype=np.int64)
        N.check(N.lib().pk_merge_shards(self._h, N.ptr(blocks), int(R), int(B), int(kk), N.ptr(ids),
                                        N.ptr(dd), N.ptr(cids), N.ptr(cnt), N.ptr(sc), 0))
        return ids, dd, cids, cnt, sc

    def merge_shards_device(self, blocks, R: int, B: int, kk: int, out_ids, out_d, out_cid, out_n,
                            out_scanned=None):
        N.check(N.lib().pk_merge_shards(self._h, N.ptr(blocks), int(R), int(B), int(kk),
                                        N.ptr(out_ids), N.ptr(out_d), N.ptr(out_cid), N.ptr(out_n),
                                        N.ptr(out_scanned), N.PK_DEVICE_PTRS))

    def assign(self, X, scope_code: int):
        self.flush()
        X = N.f32(X, self.dimension)
        n = X.shape[0]
        cid = np.empty(n, dtype=np.int64)
        dist = np.empty(n, dtype=np.float32)
        if n:
            N.check(N.lib().pk_assign(self._h, N.ptr(X), n, int(scope_code), N.ptr(cid),
                                      N.ptr(dist), 0))
        return cid, dist
