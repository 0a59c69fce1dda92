"""Snapshot / restore of a whole Store (ref/persist.py:136-380), in the
reference's own file format so snapshots move between the two packages.

Layout: the PNCK header and cluster records (pnck.py), then the reference's
tagged JSON sections in its order -- CMET (cluster identity, scope, delta,
centroid, counters), STAG (staged items), PAYL (payloads), GRPH (per-scope
graphs and portal pairs), PROF (scan profiles), FSMT (pattern tables), CACH
(L0 / L1 pools, window, counters), SEQS (request sequences), TIER (hotset
clock and frequencies), META (seed, id / op counters, agents, RNG state),
CONF (the StoreConfig fields the reference has).  JSON is written with sorted
keys and no whitespace and vectors as base64 of their raw f32 bytes, so a
snapshot is bit-exact across identical runs (ref tests/test_persist.py:45-49).

Restore rebuilds the device side from the records: every list is created
under its original cid with its rows in order, and the stored centroid (not a
recomputed one) is installed -- exactly the state the reference's restore
leaves (ref/persist.py:256-274); the graph is restored, not rebuilt, with the
portal adjacency rebuilt from the sorted pairs (ref/persist.py:295-299), and
the cache pools re-added item by item (ref/persist.py:313-341).  Like the
reference's restore, the L1 item -> cluster dedup index starts empty.
"""

from __future__ import annotations

import base64
import dataclasses
import json

import numpy as np

from . import pnck
from .cache import L0Entry, L1Cluster
from .clusters import Cluster
from .core import Metric, ParseError
from .fsm import AccessPatternFsm, FsmState
from .graph import _Node
from .pool import VectorPool

# StoreConfig fields of the reference (CONF carries exactly these, so the
# reference's StoreConfig(**conf) accepts our snapshots)
REFERENCE_CONFIG_FIELDS = (
    "dimension", "metric", "seed", "split_threshold", "split_target", "maintenance_interval", "n_p",
    "l0_capacity", "l1_capacity", "kappa", "alpha_et", "window_w", "verify_mode", "cache_enabled", "n_s",
    "d_merge_factor", "theta_match", "prefetch_enabled", "pattern_enabled", "m", "ef_search_factor",
    "alpha_ic", "p_size", "coarse_mode", "profiles_enabled", "accelerator", "budget_bytes", "b_insert",
    "decay_half_life", "slack_fraction", "hotset_interval", "splits_enabled", "lazy_maintenance",
    "static_writable_by_agents", "default_nprobe", "threads", "request_window")


def _b64(arr) -> str:
    return base64.b64encode(np.ascontiguousarray(arr, dtype=np.float32).tobytes()).decode()


def _unb64(s: str, dimension: int) -> np.ndarray:
    return np.frombuffer(base64.b64decode(s), dtype=np.float32).reshape(-1, dimension)[0].copy()


def _json_bytes(obj) -> bytes:
    return json.dumps(obj, sort_keys=True, separators=(",", ":")).encode()


def _key_json(key):
    return [int(x) if isinstance(x, (int, np.integer)) else x for x in key] if isinstance(key, tuple) else key


def snapshot(store, path):
    """ref/persist.py:136-241."""
    cl_store = store.clusters
    cids = sorted(cl_store.clusters)
    d = store.cfg.dimension
    records = [(cl_store.clusters[c].centroid, cl_store.clusters[c].member_ids,
                cl_store.clusters[c].vectors) for c in cids]
    sections = []

    def sec(tag, obj):
        sections.append((tag, _json_bytes(obj)))

    sec(b"CMET", {
        "clusters": [{"id": int(c), "scope": cl_store.clusters[c].scope,
                      "delta": float(cl_store.clusters[c].delta),
                      "centroid": _b64(cl_store.clusters[c].centroid),
                      "access_count": int(cl_store.clusters[c].access_count),
                      "dirty": int(cl_store.clusters[c].dirty)} for c in cids],
        "next_cid": int(cl_store._next_cid)})
    sec(b"STAG", {scope: [[int(iid), _b64(vec)] for iid, vec in items.items()]
                  for scope, items in cl_store.staged.items()})
    sec(b"PAYL", [[int(iid), base64.b64encode(p).decode()] for iid, p in sorted(store.payloads.items())])
    g = store.graph
    sec(b"GRPH", {
        "scopes": {scope: {"entry": None if sg.entry is None else int(sg.entry),
                           "max_level": int(sg.max_level),
                           "spacing_sum": float(sg.spacing_sum), "spacing_n": int(sg.spacing_n),
                           "nodes": {str(cid): {"level": int(n.level),
                                                "neighbors": [[int(x) for x in layer] for layer in n.neighbors]}
                                     for cid, n in sg.nodes.items()}}
                   for scope, sg in g.graphs.items()},
        "portal_pairs": [[int(a), int(b)] for a, b in sorted(g.portal_pairs)]})
    sec(b"PROF", [[int(c), agent, [int(x) for x in entries]]
                  for c in cids for agent, entries in cl_store.clusters[c].profiles.items()])
    sec(b"FSMT", {agent: [{"states": [{"c": _b64(s.c), "delta": float(s.delta), "hits": int(s.hits),
                                       "count": int(s.count)} for s in fsm.states],
                           "transitions": [[int(i), int(j), int(n)]
                                           for (i, j), n in sorted(fsm.transition_counts.items())],
                           "entries": [int(x) for x in fsm.entry_counts],
                           "d_merge": float(fsm.d_merge)}
                          for fsm in table.fsms]
                  for agent, table in store.patterns.items()})
    cach = {}
    for agent, cache in store.caches.items():
        cach[agent] = {
            "l0": [{"key": _key_json(key), "freq": int(e.freq), "last_access": int(e.last_access),
                    "items": [[int(iid), bool(st)] for iid, _, _, st in e.pool.rows()]}
                   for key, e in cache.l0.items()],
            "l1": [[[int(iid), bool(st)] for iid, _, _, st in cl.pool.rows()] for cl in cache.l1],
            "window": [float(x) for x in cache._window],
            "seq": int(cache._seq),
            "completed": int(cache.completed_queries),
            "verified": int(cache.verified_count),
            "miss": int(cache.miss_count)}
    sec(b"CACH", cach)
    sec(b"SEQS", {agent: [_b64(v) for v in seq] for agent, seq in store.sequences.items()})
    sec(b"TIER", {"clock": int(store.tier.clock),
                  "freq": [[int(c), float(v), int(last)] for c, (v, last) in sorted(store.tier.freq.items())],
                  "flush_count": int(store.tier.flush_count)})
    sec(b"META", {"seed": int(store.seed), "next_item_id": int(store._next_item_id),
                  "op_count": int(store._op_count), "agents": list(store.caches),
                  "rng_state": store.rng.bit_generator.state})
    cfg = store.cfg
    sec(b"CONF", {k: (getattr(cfg, k).value if isinstance(getattr(cfg, k), Metric) else getattr(cfg, k))
                  for k in REFERENCE_CONFIG_FIELDS})
    pnck.write_pnck(path, d, store.metric, records, sections)


def restore(store_cls, path, **overrides):
    """ref/persist.py:244-380; ``overrides``: StoreConfig fields of this
    package the file does not carry (``device``, ``sharded``)."""
    dimension, metric, records, sections = pnck.read_pnck(path, with_sections=True)

    def sec(tag: bytes):
        if tag not in sections:
            raise ParseError(f"missing section {tag!r}", 0)
        return json.loads(sections[tag].decode())

    from .engine import StoreConfig  # local import avoids a cycle

    conf = sec(b"CONF")
    known = {f.name for f in dataclasses.fields(StoreConfig)}
    cfg = StoreConfig(**{k: v for k, v in conf.items() if k in known}, **overrides)
    store = store_cls(cfg)
    meta = sec(b"META")
    cmeta = sec(b"CMET")
    for agent in meta["agents"]:
        store.register_agent(agent)

    cs = store.clusters
    index = store.index
    # clusters under their original ids, rows in order, the stored centroids
    for (cent, ids, mat), info in zip(records, cmeta["clusters"]):
        cid, scope = int(info["id"]), info["scope"]
        if scope not in cs.by_scope:
            cs.register_scope(scope)
        cl = Cluster(cid, scope, dimension)
        cl._metric = store.metric
        cl._host_add_many(np.asarray(ids, dtype=np.int64), mat)
        for iid in np.asarray(ids).tolist():
            cs.owner[int(iid)] = ("cluster", cid)
        centroid = _unb64(info["centroid"], dimension)
        index.create_list(cid, store.scope_codes.intern(scope), mat, ids)
        index.set_centroid(cid, centroid)
        cl.centroid = centroid
        cl.delta = info["delta"]
        cl.access_count = info["access_count"]
        cl.dirty = info["dirty"]
        cs.clusters[cid] = cl
        cs.by_scope.setdefault(scope, {})[cid] = None
    cs._next_cid = cmeta["next_cid"]

    for scope, items in sec(b"STAG").items():
        cs.register_scope(scope)
        for iid, b in items:
            cs.stage_item(scope, int(iid), _unb64(b, dimension))

    for iid, b in sec(b"PAYL"):
        store.payloads[int(iid)] = base64.b64decode(b)

    graph = store.graph
    grph = sec(b"GRPH")
    for scope, gd in grph["scopes"].items():
        graph.register_scope(scope)
        sg = graph.graphs[scope]
        sg.entry = gd["entry"]
        sg.max_level = gd["max_level"]
        sg.spacing_sum = gd["spacing_sum"]
        sg.spacing_n = gd["spacing_n"]
        for cid_s, nd in gd["nodes"].items():
            cid = int(cid_s)
            node = _Node(cid, nd["level"])
            node.neighbors = [list(layer) for layer in nd["neighbors"]]
            sg.nodes[cid] = node
            graph.scope_of[cid] = scope
            graph.slot[cid] = index.list_slot(cid)
    for a, b in grph["portal_pairs"]:
        graph.portal_pairs.add((a, b))
        graph.portals.setdefault(a, []).append(b)
        graph.portals.setdefault(b, []).append(a)
    graph.dirty = True

    for cid, agent, entries in sec(b"PROF"):
        cs.clusters[cid].profiles[agent] = list(entries)

    for agent, fsms in sec(b"FSMT").items():
        table = store.patterns[agent]
        for fd in fsms:
            states = [FsmState(_unb64(s["c"], dimension), s["delta"], s["hits"], s["count"])
                      for s in fd["states"]]
            tc = {(i, j): n for i, j, n in fd["transitions"]}
            table.fsms.append(AccessPatternFsm(states, tc, list(fd["entries"]), fd["d_merge"]))
        table.version += 1

    code = store.scope_codes.intern
    for agent, cd in sec(b"CACH").items():
        cache = store.caches[agent]
        for ed in cd["l0"]:
            key = tuple(ed["key"]) if isinstance(ed["key"], list) else ed["key"]
            entry = L0Entry(key, VectorPool(dimension, ordered=True, rows=store.rows), ed["freq"],
                            ed["last_access"])
            for iid, staged in ed["items"]:
                info = store.get_item(iid)
                if info is None:
                    continue
                vec, _, scope = info
                entry.pool.add(iid, vec, code(scope), staged)
            cache.l0[key] = entry
        for items in cd["l1"]:
            cl = L1Cluster(dimension, store.rows)
            for iid, staged in items:
                info = store.get_item(iid)
                if info is None:
                    continue
                vec, _, scope = info
                cl.add(iid, vec, code(scope), staged)
                cache._l1_unindexed.add(iid)
            cache.l1.append(cl)
        cache._window.extend(cd["window"])
        cache._seq = cd["seq"]
        cache.completed_queries = cd["completed"]
        cache.verified_count = cd["verified"]
        cache.miss_count = cd["miss"]
        cache._l1_epoch += 1

    for agent, seq in sec(b"SEQS").items():
        store.sequences[agent] = [_unb64(b, dimension) for b in seq]
        store._drows[agent] = [None] * len(store.sequences[agent])

    tier = sec(b"TIER")
    store.tier.clock = tier["clock"]
    store.tier.freq = {cid: (v, last) for cid, v, last in tier["freq"]}
    store.tier.flush_count = tier["flush_count"]

    store._next_item_id = meta["next_item_id"]
    store._op_count = meta["op_count"]
    store.rng.bit_generator.state = meta["rng_state"]
    if store.cfg.accelerator != "none":
        store.tier.hotset_update()
    return store
