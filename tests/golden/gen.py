"""Deterministic workloads shared by the golden-fixture generator
(make_golden.py, run against the reference in the authoring container) and
the parity tests (run against this package, anywhere).

Data come from numpy's PCG64 with fixed seeds, so they regenerate bit-exactly
wherever the same numpy is installed; every fixture stores a SHA-256 of the
arrays it was made from and the tests check it before comparing.
"""

from __future__ import annotations

import hashlib

import numpy as np


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def unit_sphere(rng, n, d):
    """bench/workload.py:108-111."""
    x = rng.normal(size=(n, d))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    return x.astype(np.float32)


def partition(rng, base, nlist):
    """Deterministic IVF partition (any partition works for parity: both
    sides load the same lists).  Seeds = random rows, float64 argmin."""
    seeds = base[rng.choice(len(base), nlist, replace=False)].astype(np.float64)
    b = base.astype(np.float64)
    d2 = (b * b).sum(1)[:, None] + (seeds * seeds).sum(1)[None, :] - 2 * b @ seeds.T
    lab = np.argmin(d2, axis=1)
    lists = []
    for c in range(nlist):
        rows = np.where(lab == c)[0]
        lists.append(rows)
    return lists


# ---------------------------------------------------------------- kernels
KERNEL_CASES = [
    # (name, d, n, kind)
    ("d1", 1, 17, "normal"),
    ("d3", 3, 33, "normal"),
    ("d17", 17, 40, "normal"),
    ("d64", 64, 50, "normal"),
    ("d64_big", 64, 40, "wide"),
    ("d384", 384, 37, "unit"),
    ("d768", 768, 29, "unit"),
    ("d1024", 1024, 11, "unit"),
    ("dups", 32, 24, "dups"),
]


def kernel_case(name, d, n, kind, seed=11):
    rng = np.random.default_rng(np.random.PCG64(seed + d * 7 + n))
    if kind == "unit":
        mat = unit_sphere(rng, n, d)
        q = unit_sphere(rng, 1, d)[0]
    elif kind == "wide":
        mat = (rng.normal(size=(n, d)) * np.exp(rng.uniform(-8, 8, size=(n, d)))).astype(np.float32)
        q = (rng.normal(size=d) * np.exp(rng.uniform(-8, 8, size=d))).astype(np.float32)
    elif kind == "dups":
        base = rng.normal(size=(4, d)).astype(np.float32)
        mat = base[rng.integers(0, 4, n)]
        mat[::5] = 0.0
        q = base[1].copy()
    else:
        mat = rng.normal(size=(n, d)).astype(np.float32)
        q = rng.normal(size=d).astype(np.float32)
    cents = mat[rng.integers(0, n, max(2, n // 4))] + np.float32(0.25) * rng.normal(
        size=(max(2, n // 4), d)).astype(np.float32)
    if kind == "dups":
        cents[1] = cents[0]  # exact tie -> first centroid wins
    return q, mat, cents.astype(np.float32)


# ---------------------------------------------------------------- store traces
TRACE_SPECS = {
    # name: dict(d, n_base, nlist, n_q, n_ins, n_del, n_upd, maint, splits, agents, seed)
    "ivf_small": dict(d=32, n_base=3000, nlist=24, n_q=60, n_ins=200, n_del=40, n_upd=25,
                      maint=16, split=None, agents=2, seed=5, k=10, nprobe=4),
    "ivf_d384": dict(d=384, n_base=2500, nlist=16, n_q=40, n_ins=96, n_del=16, n_upd=8,
                     maint=32, split=None, agents=0, seed=6, k=10, nprobe=3),
    "ivf_splits": dict(d=16, n_base=600, nlist=4, n_q=40, n_ins=500, n_del=30, n_upd=20,
                       maint=24, split=(220, 100), agents=1, seed=7, k=8, nprobe=3),
}


# Traces at the reference's DEFAULT coarse ef (ef_search_factor 4, approximate
# graph traversal, ref/graph.py:321-422) with multi-scope agent graphs grown by
# splits, so portals and per-scope graphs matter; they also record
# SearchStats.coarse_computations.  Replayed against this package's graph
# traversal (pk_graph.cu); the oracle's flat store model does not cover them.
GRAPH_TRACE_SPECS = {
    "graph_hybrid": dict(d=24, n_base=4000, nlist=120, n_q=140, n_ins=1600, n_del=40, n_upd=20,
                         maint=32, split=(80, 40), agents=3, seed=8, k=10, nprobe=4, ef_factor=4,
                         record_coarse=True),
    "graph_per_agent": dict(d=24, n_base=3000, nlist=90, n_q=120, n_ins=1200, n_del=30, n_upd=20,
                            maint=32, split=(80, 40), agents=3, seed=9, k=10, nprobe=3, ef_factor=4,
                            record_coarse=True, coarse_mode="per_agent"),
    "graph_ef2": dict(d=16, n_base=2500, nlist=100, n_q=120, n_ins=800, n_del=30, n_upd=20,
                      maint=16, split=(70, 30), agents=2, seed=10, k=6, nprobe=5, ef_factor=2,
                      record_coarse=True),
}


def trace_ops(spec):
    """Deterministic op list for one trace.

    ops: ("load", scope, [row-index arrays into base])
         ("insert", agent, scope, vecs f32[m, d], explicit_ids or None)
         ("delete", agent, id)
         ("update", agent, id, vec)
         ("search", agent, scopes, q, k, nprobe)
    Ids referenced by delete/update are picked by position among the ids the
    trace has created so far (both sides assign the same ids).
    """
    d = spec["d"]
    rng = np.random.default_rng(np.random.PCG64(1000 + spec["seed"]))
    base = unit_sphere(rng, spec["n_base"], d)
    lists = partition(rng, base, spec["nlist"])
    agents = [f"agent{i}" for i in range(spec["agents"])]
    ops = [("load", "static", lists)]
    k, nprobe = spec["k"], spec["nprobe"]
    all_scopes = ["static"] + agents
    n_ins, n_del, n_upd, n_q = spec["n_ins"], spec["n_del"], spec["n_upd"], spec["n_q"]
    # interleave: batches of 8 inserts, searches, deletes, updates
    events = (["I"] * (n_ins // 8)) + (["S"] * n_q) + (["D"] * n_del) + (["U"] * n_upd)
    order = rng.permutation(len(events))
    live_guess = spec["n_base"]
    for e in (events[i] for i in order):
        if e == "I":
            tgt = rng.integers(0, len(all_scopes))
            scope = all_scopes[tgt]
            agent = scope if scope != "static" else None
            if rng.random() < 0.5:
                vecs = unit_sphere(rng, 8, d)
            else:  # near existing rows: dense regions, recomputes matter
                vecs = (base[rng.integers(0, len(base), 8)] + 0.05 * unit_sphere(rng, 8, d)).astype(np.float32)
            if rng.random() < 0.15:
                vecs[3] = vecs[2]  # duplicate vector inside a batch
            ops.append(("insert", agent, scope, vecs, None))
            live_guess += 8
        elif e == "S":
            r = rng.random()
            if r < 0.4:
                q = base[rng.integers(0, len(base))].copy()  # exact hit (distance 0)
            elif r < 0.7:
                q = (base[rng.integers(0, len(base))] + 0.01 * rng.normal(size=d)).astype(np.float32)
            else:
                q = unit_sphere(rng, 1, d)[0]
            if agents and rng.random() < 0.5:
                m = rng.integers(1, len(all_scopes) + 1)
                scopes = sorted(rng.choice(all_scopes, m, replace=False).tolist())
            else:
                scopes = ["static"]
            kq = int(k if rng.random() < 0.8 else rng.integers(1, 33))
            npq = int(nprobe if rng.random() < 0.8 else rng.integers(1, spec["nlist"] + 2))
            ops.append(("search", None, scopes, q, kq, npq))
        elif e == "D":
            ops.append(("delete", None, int(rng.integers(0, live_guess))))
        else:
            v = unit_sphere(rng, 1, d)[0]
            ops.append(("update", None, int(rng.integers(0, live_guess)), v))
    # tail: exhaustive-edge search on a tiny scope and an all-scope sweep
    for i in range(4):
        ops.append(("search", None, all_scopes, unit_sphere(rng, 1, d)[0], k, nprobe))
    return base, ops


def store_config_kwargs(spec):
    """Reference StoreConfig for bare-path parity."""
    kw = dict(
        dimension=spec["d"], seed=spec["seed"], ef_search_factor=spec.get("ef_factor", 1 << 20),
        alpha_et=0.0, cache_enabled=False, pattern_enabled=False, prefetch_enabled=False,
        profiles_enabled=False, accelerator="none", maintenance_interval=spec["maint"],
        coarse_mode=spec.get("coarse_mode", "hybrid"),
    )
    if spec["split"] is None:
        kw.update(split_threshold=1 << 30, split_target=1 << 20, splits_enabled=False)
    else:
        kw.update(split_threshold=spec["split"][0], split_target=spec["split"][1], splits_enabled=True)
    return kw


def bulk_case(seed=21):
    rng = np.random.default_rng(np.random.PCG64(seed))
    n, d = 1500, 16
    centers = unit_sphere(rng, 6, d)
    x = (centers[rng.integers(0, 6, n)] + 0.2 * rng.normal(size=(n, d))).astype(np.float32)
    x[7] = x[3]  # duplicate rows
    qs = unit_sphere(rng, 20, d)
    return x, qs


# ---------------------------------------------------------------- agent-mode traces
AGENT_TRACE_SPECS = {
    # per-agent caches (small L0 / L1 so evictions, write-backs and merge-downs
    # happen), staged agent inserts, early termination (short window), FSM
    # pattern hints, prefetch, profiles, request boundaries, verify mode
    "agents_small": dict(d=24, n_base=1500, nlist=12, n_agents=2, n_ops=260, seed=31, k=5,
                         nprobe=3, n_p=4, l0=8, l1=24, window=6, alpha=0.7, verify=False),
    "agents_verify": dict(d=16, n_base=900, nlist=8, n_agents=3, n_ops=220, seed=32, k=4,
                          nprobe=2, n_p=3, l0=6, l1=16, window=4, alpha=0.9, verify=True),
    "agents_ip": dict(d=32, n_base=1200, nlist=10, n_agents=2, n_ops=240, seed=33, k=6,
                      nprobe=3, n_p=4, l0=8, l1=20, window=6, alpha=0.7, verify=False,
                      metric="ip"),
    # (no cosine agent trace: the reference raises ZeroDivisionError once an L1
    # pool empties -- its zero centroid has no cosine distance, ref/core.py:106-109)
    "agents_many": dict(d=48, n_base=3000, nlist=24, n_agents=5, n_ops=700, seed=35, k=8,
                        nprobe=4, n_p=6, l0=12, l1=40, window=8, alpha=0.6, verify=False),
    # the coordinated multi-agent shape of configs[2] scaled to the reference's
    # CPU speed: 16 agents, k 10, mixed insert / search stream
    "agents_16": dict(d=64, n_base=6000, nlist=24, n_agents=16, n_ops=1600, seed=36, k=10,
                      nprobe=4, n_p=8, l0=16, l1=64, window=8, alpha=0.7, verify=False),
    # agent mode at the reference's default coarse ef (graph traversal, portals
    # from merged-down agent clusters), coarse_computations recorded
    "agents_graph": dict(d=32, n_base=4000, nlist=80, n_agents=4, n_ops=900, seed=37, k=8,
                         nprobe=3, n_p=6, l0=10, l1=30, window=6, alpha=0.7, verify=True,
                         ef_factor=4, record_coarse=True),
}


def agent_trace_ops(spec):
    """Agent-mode op list: themed agent streams (each agent walks between a few
    centres, so patterns and cache locality exist), store-level ops mixed in.
    ops as trace_ops plus ("end_request", agent) and ("flush",)."""
    d = spec["d"]
    rng = np.random.default_rng(np.random.PCG64(2000 + spec["seed"]))
    base = unit_sphere(rng, spec["n_base"], d)
    lists = partition(rng, base, spec["nlist"])
    agents = [f"agent{i}" for i in range(spec["n_agents"])]
    themes = {a: base[rng.choice(len(base), 3, replace=False)] for a in agents}
    sigma = 0.2 * np.sqrt(2.0) / np.sqrt(d)  # bench/workload.py:73-76
    ops = [("load", "static", lists)]
    k, nprobe = spec["k"], spec["nprobe"]
    live_guess = spec["n_base"]
    step = {a: 0 for a in agents}
    for t in range(spec["n_ops"]):
        a = agents[int(rng.integers(0, len(agents)))]
        centre = themes[a][step[a] % 3]
        r = rng.random()
        if r < 0.55:
            q = (centre + sigma * rng.normal(size=d)).astype(np.float32)
            scopes = sorted([a, "static"]) if rng.random() < 0.8 else [a]
            ops.append(("search", a, scopes, q, k, nprobe))
            step[a] += 1
        elif r < 0.8:
            vecs = (centre + sigma * rng.normal(size=(int(rng.integers(1, 5)), d))).astype(np.float32)
            ops.append(("insert", a, a, vecs, None))
            live_guess += len(vecs)
        elif r < 0.86:
            ops.append(("end_request", a))
        elif r < 0.91:
            ops.append(("delete", None, int(rng.integers(0, live_guess))))
        elif r < 0.95:
            ops.append(("update", None, int(rng.integers(0, live_guess)),
                        unit_sphere(rng, 1, d)[0]))
        elif r < 0.98:
            q = unit_sphere(rng, 1, d)[0]
            ops.append(("search", None, sorted(["static"] + agents), q, k, nprobe))
        else:
            ops.append(("flush",))
    ops.append(("flush",))
    for a in agents:
        ops.append(("search", a, sorted([a, "static"]), themes[a][0], k, nprobe))
    return base, ops


def agent_store_config_kwargs(spec):
    """Reference StoreConfig of the agent traces (exhaustive coarse ef)."""
    return dict(
        dimension=spec["d"], seed=spec["seed"], ef_search_factor=spec.get("ef_factor", 1 << 20),
        metric=spec.get("metric", "sq_l2"), alpha_et=spec["alpha"], window_w=spec["window"], n_p=spec["n_p"],
        l0_capacity=spec["l0"], l1_capacity=spec["l1"], verify_mode=spec["verify"],
        cache_enabled=True, pattern_enabled=True, prefetch_enabled=True, profiles_enabled=True,
        accelerator="none", split_threshold=1 << 30, split_target=1 << 20, splits_enabled=False,
        maintenance_interval=16, threads=0,
    )


def run_agent_ops(store, spec, base, ops, write_pnck, metric, group_searches=False):
    """Apply an agent trace to a Store (the reference's or this package's --
    the same code drives both sides) and record what it returns.
    group_searches: each run of consecutive searches with the same (agent,
    scopes, k, nprobe) goes through ONE search_batch call (this package only;
    equal to the searches one by one)."""
    import os
    import tempfile

    rec = {"digest": np.array(digest(base)), "n_ops": np.array(len(ops))}
    for a in range(spec["n_agents"]):
        store.register_agent(f"agent{a}")
    batched = {}
    for i, op in enumerate(ops):
        kind = op[0]
        if group_searches and kind == "search" and i not in batched:
            key = (op[1], tuple(op[2]), op[4], op[5])
            j = i
            while j + 1 < len(ops) and ops[j + 1][0] == "search" and \
                    (ops[j + 1][1], tuple(ops[j + 1][2]), ops[j + 1][4], ops[j + 1][5]) == key:
                j += 1
            res = store.search_batch(op[1], op[2], np.stack([ops[t][3] for t in range(i, j + 1)]), op[4], op[5],
                                     want_scan_ids=True)
            batched.update({t: res[t - i] for t in range(i, j + 1)})
        if kind == "load":
            _, scope, lists = op
            with tempfile.TemporaryDirectory() as td:
                path = os.path.join(td, "base.pnck")
                write_pnck(path, spec["d"], metric,
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
        elif kind == "end_request":
            store.end_request(op[1])
        elif kind == "flush":
            store.flush_caches()
        elif kind == "search":
            _, agent, scopes, q, k, nprobe = op
            res = batched.pop(i) if group_searches else store.search(agent, scopes, q, k, nprobe)
            rec[f"{i}/hit_ids"] = np.array([h[0] for h in res.hits], dtype=np.int64)
            rec[f"{i}/hit_d"] = np.array([h[1] for h in res.hits], dtype=np.float32)
            rec[f"{i}/hit_scope"] = np.array([h[2] for h in res.hits], dtype="U16")
            rec[f"{i}/scanned"] = np.array(res.stats.scanned_vectors)
            rec[f"{i}/scan_ids"] = np.asarray(res.scan_ids, dtype=np.int64)
            rec[f"{i}/level"] = np.array(res.stats.level_reached, dtype="U4")
            rec[f"{i}/early"] = np.array(bool(res.stats.early_terminated))
            if spec.get("record_coarse"):
                rec[f"{i}/coarse"] = np.array(res.stats.coarse_computations)
    cl = store.clusters.clusters
    cids = sorted(cl)
    rec["final/cids"] = np.array(cids, dtype=np.int64)
    rec["final/scopes"] = np.array([cl[c].scope for c in cids], dtype="U16")
    rec["final/centroids"] = np.stack([cl[c].centroid for c in cids])
    rec["final/sizes"] = np.array([cl[c].size for c in cids], dtype=np.int64)
    rec["final/members"] = np.concatenate([cl[c].member_ids for c in cids])
    rec["final/live"] = np.array(store.live_count())
    rec["final/rng"] = np.array(store.rng.random())
    for a in range(spec["n_agents"]):
        name = f"agent{a}"
        c = store.caches[name]
        rec[f"final/{name}/staged"] = np.array(sorted(store.clusters.staged.get(name, {})), dtype=np.int64)
        rec[f"final/{name}/completed"] = np.array(c.completed_queries)
        rec[f"final/{name}/verified"] = np.array(c.verified_count)
        rec[f"final/{name}/misses"] = np.array(c.miss_count)
        rec[f"final/{name}/l0_sizes"] = np.array([len(e.pool) for e in c.l0.values()], dtype=np.int64)
        rec[f"final/{name}/l1_sizes"] = np.array([len(x) for x in c.l1], dtype=np.int64)
        rec[f"final/{name}/n_fsms"] = np.array(len(store.patterns[name].fsms))
    return rec
