"""List-sharded IVF over the GPUs of one box.

The reference is single-process (ref/engine.py:141-209 builds one
``ClusterStore``); the drop-in keeps that API on one GPU and adds this layer
for configs[3] (10M x 768 over 2/4/8 B200).  Posting lists are independent
units, so the path shards without a data-path collective except ONE exchange:

1. placement: lists go to ranks by size-balanced greedy packing
   (:func:`place_lists`, deterministic -- every rank computes the same map);
2. the centroid table is replicated: each owner computes its lists' centroids
   on its device (``Cluster.recompute_stats`` arithmetic, ref/clusters.py:111-118)
   and the table is all-gathered, so every rank evaluates the identical coarse
   quantizer (ref/graph.py:321-396 at exhaustive ef) and the identical probe set;
3. each rank scans only the probed lists it owns and writes its per-query
   top-kk as one *shard result block* (layout: ``pk_shard_block_bytes`` in
   include/pancake_b200.h);
4. the blocks are all-gathered (NCCL over NVLink on GPUs, gloo in the CPU tests)
   and merged by (distance, id) with first occurrence per id
   (ref/engine.py:406-426) -- the k smallest of a union lie in the union of the
   parts' k smallest, so the merge reproduces the single-index answer exactly.

``scanned_vectors`` is the sum over shards of the rows each scanned, which is
the single-index count (every probed list is scanned by exactly its owner).
"""

from __future__ import annotations

from collections.abc import Callable, Sequence

import numpy as np

from .core import UsageError
from .index import DeviceIndex, SearchOutput


# ---------------------------------------------------------------- block layout
def block_offsets(B: int, kk: int) -> dict:
    """Byte offsets of one shard result block (mirrors pk_shard_block_bytes)."""
    nkk = int(B) * int(kk)
    o = {"ids": 0, "cids": 8 * nkk, "scanned": 16 * nkk, "dists": 16 * nkk + 8 * B,
         "n": 20 * nkk + 8 * B}
    o["total"] = (20 * nkk + 12 * B + 15) // 16 * 16
    return o


def block_views(blk: np.ndarray, B: int, kk: int):
    """(ids i64[B,kk], cids i64[B,kk], scanned i64[B], dists f32[B,kk], n i32[B])
    views into a host block."""
    o = block_offsets(B, kk)
    nkk = B * kk

    def v(key, dt, count, shape):
        return blk[o[key]:o[key] + count * np.dtype(dt).itemsize].view(dt).reshape(shape)

    return (v("ids", np.int64, nkk, (B, kk)), v("cids", np.int64, nkk, (B, kk)),
            v("scanned", np.int64, B, (B,)), v("dists", np.float32, nkk, (B, kk)),
            v("n", np.int32, B, (B,)))


# ---------------------------------------------------------------- placement
def place_lists(sizes: Sequence[int], world: int) -> np.ndarray:
    """Size-balanced greedy packing: lists in descending size (ties: lower
    index first) each go to the least-loaded rank (ties: lower rank).
    Deterministic, so every rank derives the same owner map."""
    sizes = np.asarray(sizes, dtype=np.int64)
    if world < 1:
        raise UsageError("world size must be >= 1")
    owner = np.zeros(len(sizes), dtype=np.int64)
    if world == 1 or len(sizes) == 0:
        return owner
    load = np.zeros(world, dtype=np.int64)
    order = np.lexsort((np.arange(len(sizes)), -sizes))
    for i in order:
        r = int(np.argmin(load))  # first minimum -> lowest rank on ties
        owner[i] = r
        load[r] += max(int(sizes[i]), 1)
    return owner


# ---------------------------------------------------------------- the shard
class ShardedIndex:
    """One rank's shard of a list-partitioned IVF.

    ``group`` is a ``torch.distributed`` process group (None = the default
    group when initialised, else a single process).  ``local`` is the per-rank
    index -- a :class:`DeviceIndex` on ``device`` by default (the product
    path); the CPU tests pass an oracle-backed stand-in with the same methods
    to exercise placement, replication and exchange under gloo.
    """

    def __init__(self, dimension: int, metric_code: int = 0, device: int = 0, group=None,
                 local=None, reserve_rows: int = 0, reserve_lists: int = 0):
        import torch
        import torch.distributed as dist

        self.dimension = int(dimension)
        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.group = group
        if self.dist is not None:
            self.rank = self.dist.get_rank(group)
            self.world = self.dist.get_world_size(group)
            backend = self.dist.get_backend(group)
        else:
            self.rank, self.world, backend = 0, 1, None
        self.comm_device = (torch.device("cuda", device) if backend == "nccl"
                            else torch.device("cpu"))
        self.local = local if local is not None else DeviceIndex(
            dimension, metric_code, device, reserve_rows=reserve_rows, reserve_lists=reserve_lists)
        self.owner: dict[int, int] = {}
        self.dirty: dict[int, int] = {}  # rows appended per list since its last maintenance

    # ---- exchange -------------------------------------------------------
    def _all_gather(self, t):
        """All-gather equal-shaped tensors (rank order) -> [world, *t.shape]."""
        import torch

        if self.world == 1:
            return t.unsqueeze(0)
        t = t.to(self.comm_device).contiguous()
        flat = t.reshape(-1)
        out = torch.empty(self.world * flat.numel(), dtype=t.dtype, device=self.comm_device)
        self.dist.all_gather_into_tensor(out, flat, group=self.group)
        return out.view(self.world, *t.shape)

    # ---- build ----------------------------------------------------------
    def load(self, cids: Sequence[int], scopes: Sequence[int], sizes: Sequence[int],
             fetch: Callable[[int], tuple], owners: Sequence[int] | None = None) -> np.ndarray:
        """Place the global lists (``cids[i]`` in scope ``scopes[i]`` with
        ``sizes[i]`` rows); ``fetch(i) -> (rows f32[n,d], ids i64[n])`` is
        called only for the lists this rank owns.  Returns the owner map
        (``owners`` overrides place_lists, e.g. data already partitioned).

        Owners compute their lists' centroids, the table is all-gathered, and
        every rank then registers the lists in GLOBAL order (own lists with
        rows, the others centroid-only), so list handles -- the slot indices
        the dispatch path exchanges -- agree on every rank."""
        import torch

        cids = np.asarray(cids, dtype=np.int64)
        scopes = np.asarray(scopes, dtype=np.int64)
        owners = (place_lists(sizes, self.world) if owners is None
                  else np.asarray(owners, dtype=np.int64))
        mine = np.nonzero(owners == self.rank)[0]
        d = self.dimension
        data = {}
        cent_mine = np.zeros((len(mine), d), dtype=np.float32)
        for j, i in enumerate(mine):
            rows, ids = fetch(int(i))
            data[int(i)] = (rows, ids)
            cent_mine[j] = self.local.centroid_of(rows)
        # rank r's lists are exactly owners == r in index order: only the
        # padded centroid rows travel
        counts = np.bincount(owners, minlength=self.world)
        cmax = int(counts.max()) if len(counts) else 0
        pad = np.zeros((max(cmax, 1), d), dtype=np.float32)
        pad[:len(mine)] = cent_mine
        allc = self._all_gather(torch.from_numpy(pad)).cpu().numpy()
        pos = np.zeros(len(cids), dtype=np.int64)
        for r in range(self.world):
            w = np.nonzero(owners == r)[0]
            pos[w] = np.arange(len(w))
        for i in range(len(cids)):
            if owners[i] == self.rank:
                rows, ids = data.pop(int(i))
                self.local.create_list(int(cids[i]), int(scopes[i]), rows, ids)
            else:
                self.local.add_remote_list(int(cids[i]), int(scopes[i]), allc[owners[i], pos[i]])
        self.owner = {int(c): int(o) for c, o in zip(cids, owners)}
        return owners

    # ---- inserts ------------------------------------
    def insert(self, X, ids, scope_code: int, maintenance_interval: int = 256) -> np.ndarray:
        """Insert a batch that every rank receives (the ``agent=None`` path,
        ref/engine.py:571-605 / 647-660): each vector goes to the nearest
        in-scope list (assign_nearest, ref/clusters.py:268-279; ties -> lower
        cid), computed identically on every rank from the replicated
        centroids; the owner appends the row (Cluster.add).  When a list's
        dirty count reaches ``maintenance_interval`` its owner recomputes the
        centroid (fp64 row-order mean, ref/clusters.py:111-118, 294-299), the
        new centroid is broadcast and every rank applies it before the next
        vector is assigned -- the same op index everywhere, so the sharded
        index stays equal to the single-GPU one.  Returns the assigned cids."""
        import torch

        X = np.ascontiguousarray(X, dtype=np.float32).reshape(-1, self.dimension)
        ids = np.ascontiguousarray(ids, dtype=np.int64).reshape(-1)
        if len(ids) != len(X):
            raise ValueError("one id per row")
        n = len(X)
        out = np.empty(n, dtype=np.int64)
        i = 0
        while i < n:
            cid, _ = self.local.assign(X[i:], scope_code)
            j, fired = i, None
            while j < n:  # up to (and including) the vector whose insert triggers maintenance
                c = int(cid[j - i])
                out[j] = c
                self.dirty[c] = self.dirty.get(c, 0) + 1
                j += 1
                if self.dirty[c] >= maintenance_interval:
                    fired = c
                    break
            for k in range(i, j):
                c = int(out[k])
                if self.owner.get(c) == self.rank:
                    self.local.append(c, X[k:k + 1], ids[k:k + 1])
            if fired is not None:
                src = self.owner[fired]
                cent = np.zeros(self.dimension, dtype=np.float32)
                if src == self.rank:
                    cent = np.asarray(self.local.recompute(fired), dtype=np.float32)
                if self.world > 1:
                    t = torch.from_numpy(cent).to(self.comm_device)
                    g_src = src if self.group is None else self.dist.get_global_rank(self.group, src)
                    self.dist.broadcast(t, g_src, group=self.group)
                    cent = t.cpu().numpy()
                if src != self.rank:
                    self.local.set_centroid(fired, cent)
                self.dirty[fired] = 0
            i = j
        return out

    # ---- search ---------------------------------------------------------
    def search(self, Q, scope_codes, nprobe: int, kk: int) -> SearchOutput:
        """Host path: local scan -> all-gather of the shard blocks -> merge."""
        import torch

        Q = np.ascontiguousarray(Q, dtype=np.float32).reshape(-1, self.dimension)
        B = Q.shape[0]
        blk = self.local.search_block(Q, scope_codes, nprobe, kk)
        if self.world == 1:
            blocks = blk
        else:
            blocks = self._all_gather(torch.from_numpy(blk)).cpu().numpy().reshape(-1)
        ids, dd, cids, cnt, sc = self.local.merge_shards(blocks, self.world, B, kk)
        return SearchOutput(ids, dd, cids, cnt, None, sc)

    def search_device(self, Q, scope_codes, nprobe: int, kk: int, block, gathered, out_ids,
                      out_d, out_cid, out_n, out_scanned=None):
        """Device path (tensors on this rank's GPU, ordered on the index
        stream): local scan into ``block``, NCCL all-gather into ``gathered``
        ([world * block_bytes] uint8), device merge into the outputs.  The
        caller runs it under ``torch.cuda.stream(index stream)`` so the
        collective is ordered after the scan."""
        B = int(Q.shape[0])
        self.local.search_block_device(Q, scope_codes, nprobe, kk, block)
        if self.world > 1:
            self.dist.all_gather_into_tensor(gathered, block, group=self.group)
            src = gathered
        else:
            src = block
        self.local.merge_shards_device(src, self.world, B, kk, out_ids, out_d, out_cid, out_n,
                                       out_scanned)

    # ---- dispatch / combine: every rank brings its own batch --------------
    def search_dispatch(self, Q, scope_codes, nprobe: int, kk: int) -> SearchOutput:
        """Host path of the dispatch/combine step (weak scaling: each rank
        serves its own B queries against the whole sharded index).

        1. coarse stage on the rank's own queries (replicated centroids);
        2. all-gather of the queries and their list handles (dispatch);
        3. every rank scans its own lists for all world*B queries, one shard
           result block per origin rank;
        4. all-to-all returns each origin its blocks (combine), merged by
           (distance, id) into the rank's answers."""
        import torch

        Q = np.ascontiguousarray(Q, dtype=np.float32).reshape(-1, self.dimension)
        B = Q.shape[0]
        probe = self.local.search_coarse(Q, scope_codes, nprobe)
        if self.world == 1:
            blocks = self.local.search_probed(Q, probe, kk, B)
        else:
            Qa = self._all_gather(torch.from_numpy(Q)).cpu().numpy().reshape(-1, self.dimension)
            Pa = self._all_gather(torch.from_numpy(probe)).cpu().numpy().reshape(-1, nprobe)
            send = torch.from_numpy(self.local.search_probed(Qa, Pa, kk, B)).to(self.comm_device)
            recv = torch.empty_like(send)
            self.dist.all_to_all_single(recv, send, group=self.group)
            blocks = recv.cpu().numpy()
        ids, dd, cids, cnt, sc = self.local.merge_shards(blocks, self.world, B, kk)
        return SearchOutput(ids, dd, cids, cnt, None, sc)

    def search_dispatch_device(self, Q, scope_codes, nprobe: int, kk: int, bufs: dict,
                               out_ids, out_d, out_cid, out_n, out_scanned=None):
        """Device path of search_dispatch (tensors on this rank's GPU; run
        under ``torch.cuda.stream(index stream)``).  ``bufs`` holds the
        preallocated exchange buffers: probe [B, nprobe] i32, q_all
        [world*B, d] f32, probe_all [world*B, nprobe] i32, send / recv
        [world * block_bytes(B, kk)] u8."""
        B = int(Q.shape[0])
        self.local.search_coarse_device(Q, scope_codes, nprobe, bufs["probe"])
        if self.world > 1:
            self.dist.all_gather_into_tensor(bufs["q_all"], Q, group=self.group)
            self.dist.all_gather_into_tensor(bufs["probe_all"], bufs["probe"], group=self.group)
            self.local.search_probed_device(bufs["q_all"], bufs["probe_all"], kk, B, bufs["send"])
            self.dist.all_to_all_single(bufs["recv"], bufs["send"], group=self.group)
            src = bufs["recv"]
        else:
            self.local.search_probed_device(Q, bufs["probe"], kk, B, bufs["send"])
            src = bufs["send"]
        self.local.merge_shards_device(src, self.world, B, kk, out_ids, out_d, out_cid, out_n,
                                       out_scanned)

    # ---- fused combine over peer memory ----------------------------------------
    def setup_peer_combine(self, B: int, kk: int):
        """Map every rank's receive area into this process (CUDA IPC handles
        exchanged over the process group); afterwards search_dispatch_device
        can combine by P2P stores instead of an all-to-all."""
        handle = self.local.combine_create(self.world, self.rank, B, kk)
        if self.world > 1:
            handles = [None] * self.world
            self.dist.all_gather_object(handles, handle, group=self.group)
            for r, h in enumerate(handles):
                if r != self.rank:
                    self.local.combine_open(r, handle=h)
        self._epoch = 0

    def search_dispatch_peer(self, Q, scope_codes, nprobe: int, kk: int, bufs: dict, out_ids,
                             out_d, out_cid, out_n, out_scanned=None):
        """search_dispatch_device with the combine fused into the scan's
        write-out: results go straight into their origin rank's HBM (P2P) and
        the merge waits on device-side flags -- no all-to-all."""
        self._epoch += 1
        self.local.search_coarse_device(Q, scope_codes, nprobe, bufs["probe"])
        if self.world > 1:
            self.dist.all_gather_into_tensor(bufs["q_all"], Q, group=self.group)
            self.dist.all_gather_into_tensor(bufs["probe_all"], bufs["probe"], group=self.group)
            qa, pa = bufs["q_all"], bufs["probe_all"]
        else:
            qa, pa = Q, bufs["probe"]
        self.local.combine_search_probed_device(qa, pa, self._epoch)
        self.local.combine_merge_device(self._epoch, out_ids, out_d, out_cid, out_n, out_scanned)



# ---------------------------------------------------------------- Store behind the shards
class ShardedStoreIndex:
    """The device index of a ``Store`` whose clusters AND agents are sharded
    over the ranks of a process group (BASELINE north_star: "clusters and
    agents are sharded across the 8 GPUs of one box").

    Every rank runs the same Store (SPMD: the same API calls in the same
    order), so the host side -- cluster bookkeeping, the coarse graph's RNG
    draws, caches, hotset policy -- is replicated and stays identical; only
    the posting-list ROWS are partitioned, each list living in the HBM of
    one owner rank:

    * agent scopes are co-located: every list of agent scope code ``c`` lives
      on rank ``(c - 1) % world`` (agents in registration order round-robin);
    * static lists go to the rank holding the fewest rows at creation
      (ties: lowest rank) -- greedy size balancing as lists arrive;
    * centroids are replicated: the owner computes a list's centroid (create,
      maintenance) and broadcasts it, so every rank's coarse quantizer and
      ``assign_nearest`` see the same table;
    * a batched search scans each rank's own probed lists into one shard
      result block, the blocks are all-gathered and merged by
      (distance, id) -- the single-index answer (the k smallest of a union
      lie in the union of the parts' k smallest);
    * the per-query pipeline's exact per-list scans (``scan_lists``) are run
      by the owners and exchanged.

    Implements the ``DeviceIndex`` methods the Store / ClusterStore /
    TierManager call."""

    def __init__(self, dimension: int, metric_code: int, device: int, group=None):
        self.sh = ShardedIndex(dimension, metric_code, device, group=group)
        self.local = self.sh.local
        self.rank, self.world = self.sh.rank, self.sh.world
        self.dimension = int(dimension)
        self.device = self.local.device
        self.owner: dict[int, int] = {}
        self.nrows: dict[int, int] = {}  # rows per list (host bookkeeping, identical on all ranks)
        self.rows_on = np.zeros(self.world, dtype=np.int64)

    # ---- placement / replication ------------------------------------------------
    def _place(self, scope_code: int, n: int) -> int:
        if scope_code != 0:
            return (int(scope_code) - 1) % self.world
        return int(np.argmin(self.rows_on))  # first minimum: lowest rank on ties

    def _bcast_centroid(self, src: int, cent) -> np.ndarray:
        import torch

        c = np.zeros(self.dimension, dtype=np.float32) if cent is None else np.asarray(cent, np.float32)
        if self.world > 1:
            t = torch.from_numpy(c.copy()).to(self.sh.comm_device)
            g = src if self.sh.group is None else self.sh.dist.get_global_rank(self.sh.group, src)
            self.sh.dist.broadcast(t, g, group=self.sh.group)
            c = t.cpu().numpy()
        return c

    def owner_of(self, cid: int) -> int:
        return self.owner[int(cid)]

    # ---- posting lists ---------------------------------------------------------
    def create_list(self, cid: int, scope_code: int, rows, ids) -> np.ndarray:
        ids = np.asarray(ids, dtype=np.int64)
        r = self._place(scope_code, len(ids))
        self.owner[int(cid)] = r
        self.nrows[int(cid)] = len(ids)
        self.rows_on[r] += len(ids)
        cent = self.local.create_list(cid, scope_code, rows, ids) if r == self.rank else None
        cent = self._bcast_centroid(r, cent)
        if r != self.rank:
            self.local.add_remote_list(cid, scope_code, cent)
        return cent

    def append(self, cid: int, rows, ids):
        r = self.owner[int(cid)]
        n = len(np.asarray(ids).reshape(-1))
        self.nrows[int(cid)] += n
        self.rows_on[r] += n
        if r == self.rank:
            self.local.append(cid, rows, ids)

    def append_rows(self, cids, rows, ids):
        cids = np.asarray(cids, dtype=np.int64)
        rows = np.asarray(rows, dtype=np.float32).reshape(len(cids), self.dimension)
        ids = np.asarray(ids, dtype=np.int64)
        for c in dict.fromkeys(cids.tolist()):
            sel = np.flatnonzero(cids == c)
            self.append(c, rows[sel], ids[sel])

    def remove_row(self, cid: int, row: int):
        r = self.owner[int(cid)]
        self.nrows[int(cid)] -= 1
        self.rows_on[r] -= 1
        if r == self.rank:
            self.local.remove_row(cid, row)

    def retire(self, cid: int):
        r = self.owner.pop(int(cid))
        self.rows_on[r] -= self.nrows.pop(int(cid))
        self.local.retire(cid)

    def recompute(self, cid: int) -> np.ndarray:
        r = self.owner[int(cid)]
        cent = self.local.recompute(cid) if r == self.rank else None
        cent = self._bcast_centroid(r, cent)
        if r != self.rank:
            self.local.set_centroid(cid, cent)
        return cent

    def size(self, cid: int) -> int:
        return self.nrows[int(cid)]

    def read(self, cid: int):
        """Rows / ids of a list this rank owns."""
        if self.owner[int(cid)] != self.rank:
            raise UsageError(f"cluster {cid} lives on rank {self.owner[int(cid)]}")
        return self.local.read(cid)

    def assign(self, X, scope_code: int):
        return self.local.assign(X, scope_code)  # replicated centroids: same answer everywhere

    def coarse_cids(self, Q, scope_codes, nprobe: int):
        return self.local.coarse_cids(Q, scope_codes, nprobe)

    # ---- search ------------------------------------------------------------------
    def search(self, Q, scope_codes, nprobe: int, kk: int, want_probe: bool = False) -> SearchOutput:
        out = self.sh.search(Q, scope_codes, nprobe, kk)
        if want_probe:
            out.probe = self.local.coarse_cids(Q, scope_codes, nprobe)
        return out

    # ---- the coarse graph: replicated (every rank holds every centroid) ----
    def graph_set(self, *args):
        self.local.graph_set(*args)

    def centroid_dists(self, V):
        return self.local.centroid_dists(V)

    def list_slot(self, cid: int) -> int:
        return self.local.list_slot(cid)

    def graph_probe(self, Q, scope_codes, nprobe: int, ef: int, mode: int = 0):
        return self.local.graph_probe(Q, scope_codes, nprobe, ef, mode)

    def search_graph(self, Q, scope_codes, nprobe: int, kk: int, ef: int, mode: int = 0,
                     want_probe: bool = False):
        """pk_search_graph on every rank (identical traversal, own lists
        scanned) -> all-gather of the shard blocks -> merge."""
        import torch

        Q = np.ascontiguousarray(Q, dtype=np.float32).reshape(-1, self.dimension)
        B = Q.shape[0]
        blk, probe, coarse = self.local.search_graph_block(Q, scope_codes, nprobe, kk, ef, mode)
        if self.world > 1:
            blk = self.sh._all_gather(torch.from_numpy(blk)).cpu().numpy().reshape(-1)
        ids, dd, cids, cnt, sc = self.local.merge_shards(blk, self.world, B, kk)
        return SearchOutput(ids, dd, cids, cnt, probe if want_probe else None, sc), coarse

    def scan_lists(self, q, cids, total: int):
        """(ids, dists, prefix offsets) of every row of ``cids`` in that order:
        each owner scans its lists, the pieces are exchanged."""
        cids = [int(c) for c in cids]
        mine = [c for c in cids if self.owner[c] == self.rank]
        ids, dd, pre = self.local.scan_lists(q, mine, sum(self.nrows[c] for c in mine))
        part = {c: (ids[pre[i]:pre[i + 1]], dd[pre[i]:pre[i + 1]]) for i, c in enumerate(mine)}
        if self.world > 1:
            parts = [None] * self.world
            self.sh.dist.all_gather_object(parts, part, group=self.sh.group)
            for p in parts:
                part.update(p)
        out_ids = [part[c][0] for c in cids]
        out_d = [part[c][1] for c in cids]
        pre = np.zeros(len(cids) + 1, dtype=np.int64)
        pre[1:] = np.cumsum([len(x) for x in out_ids])
        cat = (lambda xs, dt: np.concatenate(xs) if xs else np.empty(0, dtype=dt))
        return cat(out_ids, np.int64), cat(out_d, np.float32), pre

    # ---- agent path: the row store is per rank (the policy is replicated) ----------
    def rows_put(self, slots, rows):
        self.local.rows_put(slots, rows)

    def rows_reserve(self, n):
        self.local.rows_reserve(n)

    def l1_place(self, *args, **kw):
        return self.local.l1_place(*args, **kw)

    def agent_read(self, q, puts, slots, mq=None, mx=None, scope_codes=None, nprobe: int = 0,
                   ef: int = 0, mode: int = 0, cap: int = 0):
        """pk_agent_read for the replicated rows on this rank, then the
        coarse traversal (replicated centroids) and the owners' list scans."""
        d, m, _ = self.local.agent_read(q, puts, slots, mq, mx)
        lists = None
        if nprobe > 0:
            cids, coarse = self.local.graph_probe(np.asarray(q, np.float32)[None, :], scope_codes, nprobe,
                                                  ef, mode)
            sel = [int(c) for c in cids[0] if c >= 0]
            ids, dd, pre_sel = self.scan_lists(q, sel, 0)
            pre = np.zeros(nprobe + 1, dtype=np.int64)
            pre[1:len(sel) + 1] = pre_sel[1:]
            pre[len(sel) + 1:] = pre_sel[-1]
            lists = (cids[0], int(coarse[0]), pre, ids, dd)
        return d, m, lists

    # ---- tier / lifecycle ----------------------------------------------------------
    def enable_tier(self, reserve_rows: int = 0):
        raise UsageError("the native cold tier is per GPU; a sharded Store keeps every list in HBM")

    def nbytes(self) -> int:
        return self.local.nbytes()

    def tier_stats(self) -> dict:
        return self.local.tier_stats()

    def flush(self):
        self.local.flush()

    def sync(self):
        self.local.sync()

    def close(self):
        self.local.close()
