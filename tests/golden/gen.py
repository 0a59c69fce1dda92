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
        dimension=spec["d"], seed=spec["seed"], ef_search_factor=1 << 20, alpha_et=0.0,
        cache_enabled=False, pattern_enabled=False, prefetch_enabled=False,
        profiles_enabled=False, accelerator="none", maintenance_interval=spec["maint"],
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
