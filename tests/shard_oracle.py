"""Oracle-backed stand-in for one rank's DeviceIndex (TEST INFRASTRUCTURE).

Lets the CPU suite run the sharded path's host logic -- placement, centroid
replication, block exchange over gloo, merge -- with the C oracle computing
each shard's local answer.  Same method names as DeviceIndex.
"""

from __future__ import annotations

import numpy as np

from oracle import oracle as O
from paper_2602_21477_b200.sharded import block_offsets, block_views


class OracleShard:
    def __init__(self, d: int):
        self.d = d
        self.lists = []  # (cid, scope, rows, ids, centroid)

    def create_list(self, cid, scope, rows, ids):
        rows = np.ascontiguousarray(rows, dtype=np.float32).reshape(-1, self.d)
        c = O.centroid(rows)
        self.lists.append((int(cid), int(scope), rows, np.asarray(ids, dtype=np.int64), c))
        return c

    def add_remote_list(self, cid, scope, centroid):
        self.lists.append((int(cid), int(scope), np.zeros((0, self.d), np.float32),
                           np.zeros(0, np.int64), np.asarray(centroid, np.float32)))

    def _at(self, cid):
        return next(i for i, l in enumerate(self.lists) if l[0] == int(cid))

    def assign(self, X, scope_code):
        """assign_nearest per row over the in-scope lists (ties -> lower cid)."""
        X = np.ascontiguousarray(X, dtype=np.float32).reshape(-1, self.d)
        cand = [l for l in self.lists if l[1] == int(scope_code)]
        cents = np.stack([l[4] for l in cand])
        cids = np.array([l[0] for l in cand], dtype=np.int64)
        out = np.array([O.assign_nearest(x, cents, cids) for x in X], dtype=np.int64)
        return out, np.zeros(len(X), np.float32)

    def append(self, cid, rows, ids):
        i = self._at(cid)
        c, s, r, ii, cent = self.lists[i]
        rows = np.ascontiguousarray(rows, dtype=np.float32).reshape(-1, self.d)
        self.lists[i] = (c, s, np.concatenate([r, rows]), np.concatenate([ii, np.asarray(ids, np.int64)]), cent)

    def recompute(self, cid):
        i = self._at(cid)
        c, s, r, ii, _ = self.lists[i]
        cent = O.centroid(r)
        self.lists[i] = (c, s, r, ii, cent)
        return cent

    def set_centroid(self, cid, centroid):
        i = self._at(cid)
        c, s, r, ii, _ = self.lists[i]
        self.lists[i] = (c, s, r, ii, np.asarray(centroid, np.float32).copy())

    def centroid_of(self, rows):
        return O.centroid(np.ascontiguousarray(rows, dtype=np.float32).reshape(-1, self.d))

    def _flat(self):
        lists = [(i, r) for (_, _, r, i, _) in self.lists]
        cents = np.stack([c for *_, c in self.lists])
        cids = np.array([c for c, *_ in self.lists], dtype=np.int64)
        return O.FlatIVF.from_lists(lists, cents, cids), cids

    def search_coarse(self, Q, scope_codes, nprobe):
        """List handles = positions in this shard's registration order."""
        Q = np.ascontiguousarray(Q, dtype=np.float32).reshape(-1, self.d)
        flat, cids = self._flat()
        scope = np.isin([s for _, s, *_ in self.lists], list(scope_codes)).astype(np.uint8)
        _, _, _, probe, _ = flat.search(Q, nprobe, 1, in_scope=scope)
        slot = {int(c): i for i, c in enumerate(cids)}
        return np.vectorize(lambda c: slot.get(int(c), -1), otypes=[np.int32])(probe)

    def search_probed(self, Q, probe, kk, group):
        """Scan of the probed lists held here (restated with the oracle's
        distances, lexsort by (dist, id), first occurrence per id)."""
        Q = np.ascontiguousarray(Q, dtype=np.float32).reshape(-1, self.d)
        B = len(Q)
        bb = block_offsets(group, kk)["total"]
        out = np.zeros((B // group) * bb, dtype=np.uint8)
        for g in range(B // group):
            v_ids, v_cids, v_sc, v_d, v_n = block_views(out[g * bb:(g + 1) * bb], group, kk)
            v_ids[:] = -1
            v_cids[:] = -1
            v_d[:] = np.inf
            for bl in range(group):
                b = g * group + bl
                ids, ds, cs, sc = [], [], [], 0
                for h in probe[b]:
                    if h < 0:
                        continue
                    cid, _, rows, ii, _ = self.lists[h]
                    sc += len(ii)
                    if len(ii):
                        ids.append(ii)
                        ds.append(O.distances(Q[b], rows))
                        cs.append(np.full(len(ii), cid, np.int64))
                v_sc[bl] = sc
                if not ids:
                    continue
                ids, ds, cs = np.concatenate(ids), np.concatenate(ds), np.concatenate(cs)
                w = 0
                seen = set()
                for j in np.lexsort((ids, ds)):
                    if w == kk:
                        break
                    if int(ids[j]) in seen:
                        continue
                    seen.add(int(ids[j]))
                    v_ids[bl, w], v_d[bl, w], v_cids[bl, w] = ids[j], ds[j], cs[j]
                    w += 1
                v_n[bl] = w
        return out

    def search_block(self, Q, scope_codes, nprobe, kk):
        Q = np.ascontiguousarray(Q, dtype=np.float32).reshape(-1, self.d)
        B = len(Q)
        lists = [(i, r) for (_, _, r, i, _) in self.lists]
        cents = np.stack([c for *_, c in self.lists])
        cids = np.array([c for c, *_ in self.lists], dtype=np.int64)
        scope = np.isin([s for _, s, *_ in self.lists], list(scope_codes)).astype(np.uint8)
        flat = O.FlatIVF.from_lists(lists, cents, cids)
        ids, dd, cnt, _, sc = flat.search(Q, nprobe, kk, in_scope=scope)
        id2cid = {int(i): c for (c, _, _, ii, _) in self.lists for i in ii}
        blk = np.zeros(block_offsets(B, kk)["total"], dtype=np.uint8)
        v_ids, v_cids, v_sc, v_d, v_n = block_views(blk, B, kk)
        v_ids[:] = ids
        v_d[:] = dd
        v_n[:] = cnt
        v_sc[:] = sc
        v_cids[:] = np.vectorize(lambda i: id2cid.get(int(i), -1), otypes=[np.int64])(ids)
        return blk

    @staticmethod
    def merge_shards(blocks, R, B, kk):
        bb = block_offsets(B, kk)["total"]
        parts = [block_views(np.ascontiguousarray(blocks[r * bb:(r + 1) * bb]), B, kk)
                 for r in range(R)]
        return merge_reference(parts, B, kk)


def merge_reference(parts, B, kk):
    """np.lexsort((ids, dists)) + first occurrence per id (ref/engine.py:411-418)."""
    ids = np.full((B, kk), -1, np.int64)
    dd = np.full((B, kk), np.inf, np.float32)
    cids = np.full((B, kk), -1, np.int64)
    cnt = np.zeros(B, np.int32)
    sc = np.zeros(B, np.int64)
    for b in range(B):
        ci, cd, cc = [], [], []
        for (p_ids, p_cids, p_sc, p_d, p_n) in parts:
            n = int(p_n[b])
            ci.append(p_ids[b, :n])
            cd.append(p_d[b, :n])
            cc.append(p_cids[b, :n])
            sc[b] += p_sc[b]
        ci, cd, cc = np.concatenate(ci), np.concatenate(cd), np.concatenate(cc)
        order = np.lexsort((ci, cd))
        seen, w = set(), 0
        for j in order:
            if w == kk:
                break
            if int(ci[j]) in seen:
                continue
            seen.add(int(ci[j]))
            ids[b, w], dd[b, w], cids[b, w] = ci[j], cd[j], cc[j]
            w += 1
        cnt[b] = w
    return ids, dd, cids, cnt, sc
