"""CPU restatement of the reference Store's bare IVF path, on the C oracle.

TEST INFRASTRUCTURE ONLY (parity checker).  Restates, with the oracle
kernels (pancake_oracle.c) doing every distance / assignment / mean:

  load_external_ivf          ref/persist.py:397-424 (centroids recomputed)
  insert (direct place)      ref/engine.py:571-605, 647-660
  assign_nearest             ref/clusters.py:268-279
  maintenance / recompute    ref/clusters.py:111-118, 294-299
  split_cluster + k-means    ref/clusters.py:121-183, 305-350
  delete / update            ref/engine.py:680-722, ref/clusters.py:81-109, 281-292
  search (bare path)         ref/engine.py:319-426 with ref/graph.py:321-396
                             at exhaustive ef (flat top-nprobe)
  graph RNG draws            ref/graph.py:115-119, 215-237 (consumed, graph not built)

Pinned against the reference by tests/test_oracle_golden.py (the golden
traces in tests/golden were produced by the reference Store itself).
"""

from __future__ import annotations

import math

import numpy as np

from . import oracle as O


class _Cl:
    def __init__(self, cid, scope, d):
        self.id, self.scope, self.d = cid, scope, d
        self.rows = np.zeros((0, d), np.float32)
        self.ids = np.zeros(0, np.int64)
        self.centroid = np.zeros(d, np.float32)
        self.dirty = 0

    @property
    def size(self):
        return len(self.ids)


class StoreModel:
    def __init__(self, d, seed=0, maintenance_interval=256, split_threshold=1 << 30,
                 split_target=1 << 20, splits_enabled=False, metric="sq_l2"):
        self.d = d
        self.rng = np.random.default_rng(np.random.PCG64(seed))
        self.mi = maintenance_interval
        self.split_threshold = split_threshold
        self.split_target = split_target
        self.splits = splits_enabled
        self.metric = metric
        self.clusters: dict[int, _Cl] = {}
        self.by_scope: dict[str, list[int]] = {}
        self.owner: dict[int, int] = {}
        self.next_cid = 0
        self.next_id = 0
        self.nodes: dict[str, int] = {}
        self.spacing: dict[str, int] = {}
        self.register("static")

    def register(self, scope):
        self.by_scope.setdefault(scope, [])
        self.nodes.setdefault(scope, 0)
        self.spacing.setdefault(scope, 0)

    # graph.insert RNG consumption (ref/graph.py:115-119, 158-237)
    def _graph_insert(self, scope):
        while self.rng.random() < 0.5:
            pass
        if self.nodes[scope] > 0:
            self.spacing[scope] += 1
        self.nodes[scope] += 1
        if scope != "static" and self.nodes["static"] > 0 and self.spacing["static"] > 0 \
                and self.spacing[scope] > 0:
            self.rng.random()

    def create_cluster(self, scope, ids, rows):
        cid = self.next_cid
        self.next_cid += 1
        cl = _Cl(cid, scope, self.d)
        cl.ids = np.asarray(ids, np.int64).copy()
        cl.rows = np.asarray(rows, np.float32).reshape(-1, self.d).copy()
        cl.centroid = O.centroid(cl.rows)
        cl.dirty = 0
        for i in cl.ids.tolist():
            self.owner[i] = cid
        self.clusters[cid] = cl
        self.by_scope[scope].append(cid)
        self._graph_insert(scope)
        return cid

    def retire(self, cid):
        cl = self.clusters.pop(cid)
        self.by_scope[cl.scope].remove(cid)
        self.nodes[cl.scope] -= 1

    def load(self, scope, lists):
        for ids, rows in lists:
            if len(ids) == 0:
                continue
            self.create_cluster(scope, ids, rows)
            self.next_id = max(self.next_id, int(np.max(ids)) + 1)

    def _assign(self, v, scope):
        cids = self.by_scope[scope]
        cents = np.stack([self.clusters[c].centroid for c in cids])
        return O.assign_nearest(v, cents, np.array(cids), self.metric)

    def _recompute(self, cl):
        if cl.size:
            cl.centroid = O.centroid(cl.rows)
        cl.dirty = 0

    def _kmeans(self, mat, k, base_delta, max_iters=10, tol_factor=1e-4):
        """ref/clusters.py:121-183."""
        rng = self.rng
        n = len(mat)
        k = min(k, n)
        centers = np.empty((k, mat.shape[1]), np.float32)
        first = int(rng.integers(n))
        centers[0] = mat[first]
        d2 = O.sq_l2(centers[0], mat).astype(np.float64)
        for i in range(1, k):
            total = float(d2.sum())
            idx = int(rng.integers(n)) if total <= 0.0 else int(rng.choice(n, p=d2 / total))
            centers[i] = mat[idx]
            d2 = np.minimum(d2, O.sq_l2(centers[i], mat).astype(np.float64))
        js = 1e-6 * (base_delta if base_delta > 0 else 1.0)
        for i in range(1, k):
            if any(np.array_equal(centers[i], centers[j]) for j in range(i)):
                centers[i] = centers[i] + rng.normal(0.0, js, mat.shape[1]).astype(np.float32)
        labels = np.zeros(n, np.int64)
        tol = tol_factor * max(base_delta, 1e-12)
        for _ in range(max_iters):
            labels, _ = O.kmeans_assign(mat, centers)
            newc = centers.copy()
            for c in range(k):
                sel = labels == c
                if sel.any():
                    newc[c] = O.centroid(mat[sel])
                else:
                    newc[c] = mat[int(np.argmax(O.sq_l2(centers[c], mat)))]
            shift = newc - centers
            mv = float(np.max(np.sqrt(np.einsum("ij,ij->i", shift, shift))))
            centers = newc
            if mv < tol:
                break
        labels, _ = O.kmeans_assign(mat, centers)
        for c in range(k):
            if not (labels == c).any():
                counts = np.bincount(labels, minlength=k)
                donor = int(np.argmax(counts))
                labels[int(np.where(labels == donor)[0][0])] = c
        return labels

    def _delta(self, cl):
        d = O.sq_l2(cl.centroid, cl.rows)
        return float(np.mean(np.sqrt(np.maximum(d, 0.0))))

    def _split(self, cid):
        cl = self.clusters[cid]
        self._recompute(cl)
        mat, ids = cl.rows.copy(), cl.ids.copy()
        k = max(2, math.ceil(cl.size / self.split_target))
        labels = self._kmeans(mat, k, self._delta(cl))
        for c in range(int(labels.max()) + 1):
            rows = np.where(labels == c)[0]
            if len(rows):
                self.create_cluster(cl.scope, ids[rows], mat[rows])
        self.retire(cid)

    def _after_mutation(self, cid):
        cl = self.clusters[cid]
        if self.splits and cl.size >= self.split_threshold:
            self._split(cid)
        elif cl.dirty >= self.mi:
            self._recompute(cl)

    def _take_id(self, explicit=None):
        if explicit is None:
            i = self.next_id
            self.next_id += 1
            return i
        self.next_id = max(self.next_id, explicit + 1)
        return explicit

    def insert(self, scope, vecs, ids=None):
        out = []
        for i, v in enumerate(vecs):
            iid = self._take_id(None if ids is None else ids[i])
            v = np.asarray(v, np.float32)
            if not self.by_scope[scope]:
                self.create_cluster(scope, [iid], v[None])
            else:
                cid = self._assign(v, scope)
                cl = self.clusters[cid]
                cl.rows = np.concatenate([cl.rows, v[None]])
                cl.ids = np.concatenate([cl.ids, [iid]])
                cl.dirty += 1
                self.owner[iid] = cid
                self._after_mutation(cid)
            out.append(iid)
        return out

    def delete(self, iid):
        cid = self.owner.pop(iid, None)
        if cid is None:
            return False
        cl = self.clusters[cid]
        row = int(np.where(cl.ids == iid)[0][0])
        last = cl.size - 1
        if row != last:
            cl.rows[row] = cl.rows[last]
            cl.ids[row] = cl.ids[last]
        cl.rows = cl.rows[:last]
        cl.ids = cl.ids[:last]
        cl.dirty += 1
        if cl.dirty >= self.mi:
            self._recompute(cl)
        return True

    def update(self, iid, vec):
        cid = self.owner.get(iid)
        if cid is None:
            return False
        scope = self.clusters[cid].scope
        self.delete(iid)
        self.insert(scope, [vec], ids=[iid])
        return True

    def live(self):
        return len(self.owner)

    def search(self, scopes, q, k, nprobe, probe=None):
        """Returns (hits [(id, dist f32, scope)], scanned, scan_ids).  probe:
        the probed cids in coarse order when given (the coarse graph's own
        output, e.g. where it is not connected and ef cannot make it flat);
        else the flat top-nprobe by (dist, cid) (the graph at exhaustive ef,
        SURVEY F3)."""
        exhaustive = k >= self.live()
        eff = max(nprobe, len(self.clusters) or 1) if exhaustive else nprobe
        cids = [c for s in scopes for c in self.by_scope[s]]
        if not cids:
            return [], 0, np.empty(0, np.int64)
        if probe is None:
            cents = np.stack([self.clusters[c].centroid for c in cids])
            dc = O.distances(q, cents, self.metric)
            ca = np.array(cids, np.int64)
            probe = ca[np.lexsort((ca, dc))[:eff]]
        ids = [self.clusters[c].ids for c in probe]
        dd = [O.distances(q, self.clusters[c].rows, self.metric) for c in probe]
        scan_ids = np.concatenate(ids) if ids else np.empty(0, np.int64)
        if not len(scan_ids):
            return [], 0, scan_ids
        alld = np.concatenate(dd).astype(np.float32)
        order = np.lexsort((scan_ids, alld))
        hits, seen = [], set()
        for i in order:
            iid = int(scan_ids[i])
            if iid in seen:
                continue
            seen.add(iid)
            hits.append((iid, alld[i], self.clusters[self.owner[iid]].scope))
            if len(hits) >= k:
                break
        return hits, len(scan_ids), scan_ids


def bulk_build_model(x, seed, split_target):
    """Store.bulk_build (ref/engine.py:615-645) on the model."""
    m = StoreModel(x.shape[1], seed=seed)
    n = len(x)
    ids = [m._take_id() for _ in range(n)]
    k = max(1, -(-n // split_target))
    id_arr = np.asarray(ids, np.int64)
    if k == 1:
        m.create_cluster("static", id_arr, x)
        return m, ids
    center = O.centroid(x)
    spread = float(np.mean(np.sqrt(np.maximum(O.sq_l2(center, x), 0.0))))
    labels = m._kmeans(x, k, spread)
    for c in range(int(labels.max()) + 1):
        rows = np.where(labels == c)[0]
        if len(rows):
            m.create_cluster("static", id_arr[rows], x[rows])
    return m, ids
