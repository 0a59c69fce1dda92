"""The reference's hybrid coarse graph (ref/graph.py:20-422), kept on the host
exactly as the reference builds it, searched on the device.

The reference's coarse quantizer is an HNSW-style best-first traversal over
per-scope graphs of cluster centroids joined by portal edges
(``HybridGraphIndex``); at its default ``ef_search_factor`` (4) it is
approximate, so which lists a query probes -- and therefore its results --
depend on the graph's exact shape.  This module builds that shape with the
reference's algorithm and the store's shared random stream (levels, portal
coins: the same draws, so later k-means see the same stream):

* every distance it needs comes from the device in batches --
  ``DeviceIndex.centroid_dists`` returns the reference arithmetic's distance
  from a centroid to EVERY list centroid (ref/kernels.py:73-113), so one
  device call serves a whole insertion's layer searches, one more its
  neighbor-list prunings (a node's pruning reads only its own list, so the
  prunings of one insertion are independent and can be deferred);
* the structure (levels, neighbor lists in list order, portals in insertion
  order, entries, spacings) is uploaded with ``pk_graph_set`` and the search
  -- ``HybridGraphIndex.search`` / ``search_independent`` -- runs in the
  device kernel of pk_graph.cu, fused in front of the posting-list scan.
"""

from __future__ import annotations

import heapq

import numpy as np

from .core import STATIC_SCOPE, Metric, UsageError


class _Node:
    __slots__ = ("cid", "level", "neighbors")

    def __init__(self, cid: int, level: int):
        self.cid = cid
        self.level = level
        self.neighbors: list[list[int]] = [[] for _ in range(level + 1)]


class ScopeGraph:
    """One scope's layered graph (ref/graph.py:31-58)."""

    def __init__(self, scope: str):
        self.scope = scope
        self.nodes: dict[int, _Node] = {}
        self.entry: int | None = None
        self.max_level = -1
        self.spacing_sum = 0.0
        self.spacing_n = 0

    @property
    def mean_spacing(self):
        return None if self.spacing_n == 0 else self.spacing_sum / self.spacing_n

    def reset_entry(self):
        """Highest level, then lowest cid (ref/graph.py:50-58)."""
        best = None
        for cid, node in self.nodes.items():
            if best is None or (node.level, -cid) > (self.nodes[best].level, -best):
                best = cid
        self.entry = best
        self.max_level = self.nodes[best].level if best is not None else -1


def portal_probability(d_static: float, d_agent: float, alpha_ic: float) -> float:
    """ref/graph.py:61-71."""
    if d_agent <= 0.0:
        return 1.0
    return 1.0 / max(alpha_ic * d_static / d_agent, 1.0)


class _Row:
    """Distances from one centroid to every list (one device call, lazily)."""

    __slots__ = ("_g", "_vec", "_d")

    def __init__(self, g: "HybridGraph", vec):
        self._g, self._vec, self._d = g, vec, None

    def __call__(self, cid: int) -> float:
        if self._d is None:
            self._d = self._g._rows([self._vec])[0]
        return float(self._d[self._g.slot[cid]])


class HybridGraph:
    """All scopes' graphs plus portals (ref/graph.py:74-422)."""

    def __init__(self, index, centroid_of, code_of, metric: Metric, rng: np.random.Generator,
                 m: int = 16, ef_search_factor: int = 4, alpha_ic: float = 6.0,
                 ef_construction: int = 100):
        self.index = index
        self.centroid_of = centroid_of
        self.code_of = code_of  # scope name -> scope code of the device list table
        self.metric = metric
        self.rng = rng
        self.m = m
        self.ef_search_factor = ef_search_factor
        self.alpha_ic = alpha_ic
        self.ef_construction = max(ef_construction, m)
        self.graphs: dict[str, ScopeGraph] = {}
        self.portals: dict[int, list[int]] = {}
        self.portal_pairs: set[tuple[int, int]] = set()
        self.scope_of: dict[int, str] = {}
        self.slot: dict[int, int] = {}  # cid -> device list slot
        self.spacing_override: dict[str, float] = {}
        self.dirty = True

    def register_scope(self, scope: str):
        self.graphs.setdefault(scope, ScopeGraph(scope))

    def _spacing(self, scope):
        if scope in self.spacing_override:
            return self.spacing_override[scope]
        g = self.graphs.get(scope)
        return g.mean_spacing if g else None

    # ---- distances (device) ----------------------------------------------------
    def _rows(self, vecs) -> np.ndarray:
        """[len(vecs), nslots] reference distances from each vector to every
        list centroid."""
        out, _ = self.index.centroid_dists(np.stack(vecs))
        return out

    def _draw_level(self) -> int:
        level = 0
        while self.rng.random() < 0.5:
            level += 1
        return level

    @staticmethod
    def _layer_search(dist, entries, layer: int, ef: int, g: ScopeGraph):
        """ref/graph.py:125-156 (best-first in one layer of one graph)."""
        visited = {c for _, c in entries}
        cand = list(entries)
        heapq.heapify(cand)
        best = [(-d, c) for d, c in entries]
        heapq.heapify(best)
        while cand:
            d, c = heapq.heappop(cand)
            if best and d > -best[0][0] and len(best) >= ef:
                break
            node = g.nodes.get(c)
            if node is None or layer > node.level:
                continue
            for nb in node.neighbors[layer]:
                if nb in visited:
                    continue
                visited.add(nb)
                nd = dist(nb)
                if len(best) < ef or nd < -best[0][0]:
                    heapq.heappush(cand, (nd, nb))
                    heapq.heappush(best, (-nd, nb))
                    if len(best) > ef:
                        heapq.heappop(best)
        return sorted((-nd, c) for nd, c in best)

    def _prune(self, jobs):
        """Deferred neighbor-list prunings [(node, layer, candidates, keep,
        tail)]: keep the `keep` nearest of the candidates to the node's own
        centroid (ties by cid), then append `tail`."""
        if not jobs:
            return
        owners = list(dict.fromkeys(node.cid for node, *_ in jobs))
        rows = self._rows([self.centroid_of(c) for c in owners])
        at = {c: i for i, c in enumerate(owners)}
        for node, layer, cands, keep, tail in jobs:
            r = rows[at[node.cid]]
            scored = sorted((float(r[self.slot[x]]), x) for x in cands)
            node.neighbors[layer] = [x for _, x in scored[:keep]] + tail

    # ---- mutation (ref/graph.py:158-317) ------------------------------------------
    def insert(self, scope: str, cid: int) -> bool:
        g = self.graphs.get(scope)
        if g is None:
            raise UsageError(f"unknown scope {scope!r}")
        if cid in g.nodes:
            return False
        self.slot[cid] = self.index.list_slot(cid)
        self.dirty = True
        level = self._draw_level()
        node = _Node(cid, level)
        g.nodes[cid] = node
        self.scope_of[cid] = scope
        dist = _Row(self, self.centroid_of(cid))
        if g.entry is None or len(g.nodes) == 1:
            g.entry = cid
            g.max_level = level
        else:
            eps = [(dist(g.entry), g.entry)]
            for layer in range(g.max_level, level, -1):
                eps = self._layer_search(dist, eps, layer, 1, g)
            nearest = eps[0][0] if eps else None
            jobs = []
            for layer in range(min(level, g.max_level), -1, -1):
                cands = self._layer_search(dist, eps, layer, self.ef_construction, g)
                if cands:
                    nearest = cands[0][0]
                chosen = [c for _, c in sorted(cands)[:self.m]]
                node.neighbors[layer] = list(chosen)
                for nb in chosen:
                    other = g.nodes[nb]
                    if layer > other.level or cid in other.neighbors[layer]:
                        continue
                    grown = other.neighbors[layer] + [cid]
                    if len(grown) > self.m:
                        jobs.append((other, layer, grown, self.m, []))
                    else:
                        other.neighbors[layer] = grown
                eps = cands
            self._prune(jobs)
            if level > g.max_level:
                g.entry = cid
                g.max_level = level
            if nearest is not None:
                g.spacing_sum += (float(np.sqrt(max(nearest, 0.0)))
                                  if self.metric is Metric.SQUARED_EUCLIDEAN else max(nearest, 0.0))
                g.spacing_n += 1
        if scope == STATIC_SCOPE:
            return False
        return self._maybe_portal(scope, cid, dist)

    def _maybe_portal(self, scope: str, cid: int, dist) -> bool:
        """ref/graph.py:215-237."""
        static = self.graphs.get(STATIC_SCOPE)
        if static is None or static.entry is None:
            return False
        d_static, d_agent = self._spacing(STATIC_SCOPE), self._spacing(scope)
        if d_static is None or d_agent is None:
            return False
        if self.rng.random() >= portal_probability(d_static, d_agent, self.alpha_ic):
            return False
        eps = [(dist(static.entry), static.entry)]
        for layer in range(static.max_level, 0, -1):
            eps = self._layer_search(dist, eps, layer, 1, static)
        eps = self._layer_search(dist, eps, 0, 4, static)
        target = eps[0][1]
        if (cid, target) in self.portal_pairs:
            return False
        self.portal_pairs.add((cid, target))
        self.portals.setdefault(cid, []).append(target)
        self.portals.setdefault(target, []).append(cid)
        return True

    def remove(self, scope: str, cid: int):
        """ref/graph.py:239-272 (+ the orphan repair of :274-317)."""
        g = self.graphs.get(scope)
        if g is None or cid not in g.nodes:
            return
        self.dirty = True
        node = g.nodes.pop(cid)
        self.scope_of.pop(cid, None)
        jobs = []
        for other in g.nodes.values():
            for layer in range(other.level + 1):
                lst = other.neighbors[layer]
                if cid not in lst:
                    continue
                cur = [x for x in lst if x != cid]
                via = node.neighbors[layer] if layer <= node.level else []
                peers = [x for x in via if x != other.cid and x in g.nodes and x not in cur]
                if peers:
                    jobs.append((other, layer, cur + peers, self.m, []))
                else:
                    other.neighbors[layer] = cur
        self._prune(jobs)
        for other in self.portals.pop(cid, []):
            if other in self.portals:
                self.portals[other] = [x for x in self.portals[other] if x != cid]
                if not self.portals[other]:
                    del self.portals[other]
            self.portal_pairs.discard((cid, other))
            self.portal_pairs.discard((other, cid))
        if g.entry == cid:
            g.reset_entry()
        self._reconnect(g)
        self.slot.pop(cid, None)

    def _reconnect(self, g: ScopeGraph):
        if g.entry is None or len(g.nodes) <= 1:
            return

        def absorb(start, reach):
            frontier = [start]
            while frontier:
                nxt = []
                for c in frontier:
                    for nb in g.nodes[c].neighbors[0]:
                        if nb in g.nodes and nb not in reach:
                            reach.add(nb)
                            nxt.append(nb)
                frontier = nxt

        reach = {g.entry}
        absorb(g.entry, reach)
        for orphan in sorted(set(g.nodes) - reach):
            if orphan in reach:
                continue
            dist = _Row(self, self.centroid_of(orphan))
            anchor = min(reach, key=lambda r: (dist(r), r))
            an = g.nodes[anchor]
            if orphan not in an.neighbors[0]:
                grown = an.neighbors[0] + [orphan]
                if len(grown) > self.m:
                    self._prune([(an, 0, [x for x in grown if x != orphan], self.m - 1, [orphan])])
                else:
                    an.neighbors[0] = grown
            reach.add(orphan)
            absorb(orphan, reach)

    # ---- device upload ---------------------------------------------------------
    def upload(self):
        """pk_graph_set: every node's layers (M-padded, list order), portals,
        and each scope's entry / max level."""
        if not self.dirty:
            return
        M = self.m
        cids, levels, nbr, por_ptr, por = [], [], [], [0], []
        for g in self.graphs.values():
            for c, node in g.nodes.items():
                cids.append(c)
                levels.append(node.level)
                for lst in node.neighbors:
                    nbr.extend(lst)
                    nbr.extend([-1] * (M - len(lst)))
                p = self.portals.get(c, [])
                por.extend(p)
                por_ptr.append(len(por))
        codes, entries, maxl = [], [], []
        for scope, g in self.graphs.items():
            codes.append(self.code_of(scope))
            entries.append(-1 if g.entry is None else g.entry)
            maxl.append(max(g.max_level, 0))
        self.index.graph_set(M, cids, levels, nbr, por_ptr, por, self.code_of(STATIC_SCOPE), codes,
                             entries, maxl)
        self.dirty = False

    def ef_for(self, nprobe: int, ef_search: int | None = None) -> int:
        """ref/graph.py:338-340."""
        if ef_search is None:
            ef_search = self.ef_search_factor * nprobe
        return max(ef_search, nprobe)

    def node_count(self) -> int:
        return sum(len(g.nodes) for g in self.graphs.values())
