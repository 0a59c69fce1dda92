"""Replay of the golden traces (tests/golden/gen.py) against either the
oracle store model or this package's Store, producing the same record keys
as tests/golden/make_golden.py."""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
if GOLDEN not in sys.path:
    sys.path.insert(0, GOLDEN)
import gen  # noqa: E402


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def replay_model(spec):
    from oracle.store_model import StoreModel

    base, ops = gen.trace_ops(spec)
    kw = gen.store_config_kwargs(spec)
    m = StoreModel(spec["d"], seed=kw["seed"], maintenance_interval=kw["maintenance_interval"],
                   split_threshold=kw["split_threshold"], split_target=kw["split_target"],
                   splits_enabled=kw["splits_enabled"])
    for i in range(spec["agents"]):
        m.register(f"agent{i}")
    rec = {"digest": gen.digest(base)}
    for i, op in enumerate(ops):
        kind = op[0]
        if kind == "load":
            _, scope, lists = op
            m.load(scope, [(rows.astype(np.int64), base[rows]) for rows in lists])
        elif kind == "insert":
            _, agent, scope, vecs, ids = op
            rec[f"{i}/ids"] = np.array(m.insert(scope, list(vecs), ids), dtype=np.int64)
        elif kind == "delete":
            rec[f"{i}/ok"] = np.array(m.delete(op[2]))
        elif kind == "update":
            rec[f"{i}/ok"] = np.array(m.update(op[2], op[3]))
        elif kind == "search":
            _, agent, scopes, q, k, nprobe = op
            hits, scanned, scan_ids = m.search(scopes, q, k, nprobe)
            rec[f"{i}/hit_ids"] = np.array([h[0] for h in hits], dtype=np.int64)
            rec[f"{i}/hit_d"] = np.array([h[1] for h in hits], dtype=np.float32)
            rec[f"{i}/hit_scope"] = np.array([h[2] for h in hits], dtype="U16")
            rec[f"{i}/scanned"] = np.array(scanned)
            rec[f"{i}/scan_ids"] = scan_ids
    cids = sorted(m.clusters)
    rec["final/cids"] = np.array(cids, dtype=np.int64)
    rec["final/scopes"] = np.array([m.clusters[c].scope for c in cids], dtype="U16")
    rec["final/centroids"] = np.stack([m.clusters[c].centroid for c in cids])
    rec["final/sizes"] = np.array([m.clusters[c].size for c in cids], dtype=np.int64)
    rec["final/members"] = np.concatenate([m.clusters[c].ids for c in cids])
    rec["final/live"] = np.array(m.live())
    rec["final/rng"] = np.array(m.rng.random())
    return rec


def replay_store(spec, batch_searches=False, overrides=None, tier_log=None):
    """Replay on paper_2602_21477_b200.Store (needs the GPU).  ``overrides``
    change StoreConfig fields that must not change results (e.g. the native
    cold tier); ``tier_log`` collects tier metrics after every search."""
    import tempfile

    from paper_2602_21477_b200 import Store, StoreConfig
    from paper_2602_21477_b200.core import Metric
    from paper_2602_21477_b200.pnck import write_pnck

    base, ops = gen.trace_ops(spec)
    kw = gen.store_config_kwargs(spec)
    kw.update(overrides or {})
    store = Store(StoreConfig(**kw))
    for i in range(spec["agents"]):
        store.register_agent(f"agent{i}")
    rec = {"digest": gen.digest(base)}
    for i, op in enumerate(ops):
        kind = op[0]
        if kind == "load":
            _, scope, lists = op
            with tempfile.TemporaryDirectory() as td:
                path = os.path.join(td, "base.pnck")
                write_pnck(path, spec["d"], Metric.SQUARED_EUCLIDEAN,
                           [(np.zeros(spec["d"], np.float32), rows.astype(np.int64), base[rows])
                            for rows in lists])
                rec[f"{i}/count"] = np.array(store.load_external_ivf(path, scope))
        elif kind == "insert":
            _, agent, scope, vecs, ids = op
            rec[f"{i}/ids"] = np.array(store.insert(agent, scope, list(vecs), ids=ids), dtype=np.int64)
        elif kind == "delete":
            rec[f"{i}/ok"] = np.array(store.delete(op[1], op[2]))
        elif kind == "update":
            rec[f"{i}/ok"] = np.array(store.update(op[1], op[2], vector=op[3]))
        elif kind == "search":
            _, agent, scopes, q, k, nprobe = op
            if batch_searches:
                res = store.search_batch(agent, scopes, q[None], k, nprobe, want_scan_ids=True)[0]
            else:
                res = store.search(agent, scopes, q, k, nprobe)
            rec[f"{i}/hit_ids"] = np.array([h[0] for h in res.hits], dtype=np.int64)
            rec[f"{i}/hit_d"] = np.array([h[1] for h in res.hits], dtype=np.float32)
            rec[f"{i}/hit_scope"] = np.array([h[2] for h in res.hits], dtype="U16")
            rec[f"{i}/scanned"] = np.array(res.stats.scanned_vectors)
            rec[f"{i}/scan_ids"] = np.asarray(res.scan_ids, dtype=np.int64)
            rec[f"{i}/coarse"] = np.array(res.stats.coarse_computations)
            if tier_log is not None:
                tier_log.append(store.tier.metrics())
    cids = sorted(store.clusters.clusters)
    cl = store.clusters.clusters
    rec["final/cids"] = np.array(cids, dtype=np.int64)
    rec["final/scopes"] = np.array([cl[c].scope for c in cids], dtype="U16")
    rec["final/centroids"] = np.stack([cl[c].centroid for c in cids])
    rec["final/sizes"] = np.array([cl[c].size for c in cids], dtype=np.int64)
    rec["final/members"] = np.concatenate([cl[c].member_ids for c in cids])
    rec["final/live"] = np.array(store.live_count())
    rec["final/rng"] = np.array(store.rng.random())
    # device rows must mirror the host rows exactly
    owned = getattr(store.index, "owner", None)  # sharded Store: this rank's lists only
    for c in cids:
        if owned is not None and owned[c] != store.index.rank:
            continue
        rows, ids = store.index.read(c)
        assert np.array_equal(ids, cl[c].member_ids), f"device ids of cluster {c} diverged"
        assert np.array_equal(rows.view(np.uint32), cl[c].vectors.view(np.uint32)), f"device rows {c}"
    store.close()
    return rec


def compare_records(got, want, skip=("digest",)):
    """Exact comparison (float32 compared bitwise)."""
    assert str(got["digest"]) == str(want["digest"]), "workload drifted from the fixture's data"
    mism = []
    for key, w in want.items():
        if key in skip or key == "n_ops" or key.endswith("/count"):
            continue
        if key not in got:
            mism.append(f"{key}: missing")
            continue
        g = np.asarray(got[key])
        w = np.asarray(w)
        if g.dtype.kind == "f" and w.dtype.kind == "f" and g.dtype == np.float32:
            same = g.shape == w.shape and np.array_equal(g.view(np.uint32), w.astype(np.float32).view(np.uint32))
        else:
            same = g.shape == w.shape and np.array_equal(g, w)
        if not same:
            mism.append(f"{key}: got {g.tolist()[:12]} want {w.tolist()[:12]}")
    return mism
