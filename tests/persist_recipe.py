"""A store built by a fixed op sequence, probes and a continuation trace --
run against this package in-process and against the reference package
(baseline/_ref) in a subprocess, so snapshots can be compared and moved
between the two (tests/test_gpu_persist.py).

    python tests/persist_recipe.py build OUT.pnck RESULTS.json
    python tests/persist_recipe.py restore IN.pnck RESULTS.json

runs the REFERENCE package (the subprocess side).
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

D = 16


def build(Store, StoreConfig):
    """pkg/tests/test_acceptance.py:406-418's store (agent ops, splits, an
    ended request), plus a second agent."""
    store = Store(StoreConfig(dimension=D, seed=77, split_threshold=64, split_target=32))
    a = store.register_agent("a1")
    b = store.register_agent("b2")
    rng = np.random.default_rng(5)
    store.insert(None, "static", rng.normal(size=(300, D)).astype(np.float32),
                 [f"s{i}".encode() for i in range(300)])
    for i in range(40):
        v = rng.normal(size=D).astype(np.float32)
        ag = a if i % 3 else b
        store.insert(ag, ag, [v], [f"p{i}".encode()])
        store.search(ag, [ag, "static"], v, 3)
        if i % 10 == 9:
            store.end_request(ag)
    store.end_request(a)
    return store


def _res(r):
    return {"hits": [[int(h[0]), float(np.float32(h[1])).hex(), h[2]] for h in r.hits],
            "level": r.stats.level_reached, "early": bool(r.stats.early_terminated),
            "scanned": int(r.stats.scanned_vectors)}


def probes(store, n=60):
    rng = np.random.default_rng(404)
    out = []
    for _ in range(n):
        q = rng.normal(size=D).astype(np.float32)
        r = store.search(None, ["a1", "b2", "static"], q, 5, nprobe=max(len(store.clusters.clusters), 1))
        out.append(_res(r))
    return out


def continuation(store):
    """Agent traffic after a restore: cache hits and promotions, patterns,
    inserts (staged and direct), a split, deletes."""
    rng = np.random.default_rng(99)
    out = []
    themes = rng.normal(size=(3, D)).astype(np.float32)
    for i in range(60):
        ag = "a1" if i % 2 else "b2"
        v = (themes[i % 3] + 0.3 * rng.normal(size=D)).astype(np.float32)
        if i % 5 == 0:
            ids = store.insert(ag, ag, [v], [b"c"])
            out.append({"insert": [int(x) for x in ids]})
        out.append(_res(store.search(ag, [ag, "static"], v, 4)))
        if i % 7 == 6:
            ids = store.insert(None, "static", rng.normal(size=(30, D)).astype(np.float32))
            out.append({"insert_static": len(ids)})
        if i % 11 == 10:
            store.end_request(ag)
    out.append({"live": int(store.live_count()), "next_item_id": int(store._next_item_id)})
    return out


def _reference():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for src in (os.path.join(root, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(src, "agentmem")):
            sys.path.insert(0, src)
            break
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="pk_numba_"))
    import agentmem

    return agentmem.Store, agentmem.StoreConfig


if __name__ == "__main__":
    mode, path, out = sys.argv[1:4]
    Store, StoreConfig = _reference()
    if mode == "build":
        s = build(Store, StoreConfig)
        s.snapshot(path)
        res = {"probes": probes(s)}
    else:
        s = Store.restore(path)
        res = {"probes": probes(s), "continuation": continuation(s)}
    with open(out, "w") as f:
        json.dump(res, f)
