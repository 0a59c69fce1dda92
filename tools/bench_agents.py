#!/usr/bin/env python3
"""configs[2]: 16 agents x 250K x 1024 with the multi-level cache and the
coordinated index manager, mixed insert / search stream, through the public
Store API -- and the reference ``agentmem`` Store on the same host, the same
data and the same op stream (its own package, ``baseline/_ref``), so the
answers are compared op by op and the two costs are timed side by side.

    python tools/bench_agents.py [--agents 16] [--rows 250000] [--d 1024]
                                 [--rounds 8] [--batch 32] [--ref-rounds 2]

Data.  The static scope and every agent scope hold `rows` unit-sphere rows
(seeded Philox on the device), cut into IVF lists of ~2048 rows (the
reference's split_target) by nearest-seed assignment and loaded as PNCK-style
lists (``Store.load_lists`` here, ``load_external_ivf`` of the same records on
the reference side).

Stream (the reference's step-wise generator, bench/workload.py:121-140, with
an exploration share).  Every agent has G = 3 theme centres, rows of its own
scope (as the golden agent traces, tests/golden/gen.py:233-273).  One round
gives every agent one request: an insert batch of 8 near the request's first
theme (staged into the agent's cache, merged down as a base cluster when an L1
pool fills), then a search batch of `batch` queries over [agent, static] with
k 10 and nprobe 8, step j drawing near theme j mod G (sigma = 0.2 sqrt(2) /
sqrt(d), bench/workload.py:73-76) -- except a share `explore` of the steps,
which ask about a fresh random direction -- then end_request.  Revisited
themes are what the agent cache holds; the exploration queries complete at
L2 and keep the agent's distance envelope d_agent (ref/cache.py:130-150)
representative, so the early-termination rule fires on the revisits
(alpha_et 0.7) and never with alpha_et 0.

Both stores: default StoreConfig (cache, FSM patterns, prefetch, profiles,
hybrid coarse graph at ef_search_factor 4, splits on) except
accelerator="none" and threads=0 (the reference's deterministic inline mode,
so its prefetches land at the same op as ours).  Round 0 is untimed on both
sides (first-call costs, numba compilation); rounds 1.. are timed.  The
reference runs the first `ref-rounds` rounds (its cost is ~20 ms per op) and
every search result of those rounds is compared (ids, distance bits, level,
early flag, scanned count).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

G = 3


def scope_rows(torch, dev, n, d, nlist, seed):
    """Unit-sphere rows, nearest-seed lists: (rows f32[n, d] in list order,
    list lengths)."""
    g = torch.Generator(device=dev).manual_seed(seed)
    X = torch.randn(n, d, generator=g, device=dev)
    X = (X / X.norm(dim=1, keepdim=True)).float().contiguous()
    S = X[:nlist].clone()
    lab = torch.empty(n, dtype=torch.int64, device=dev)
    for s in range(0, n, 65536):
        lab[s:s + 65536] = (X[s:s + 65536] @ S.T).argmax(dim=1)
    order = torch.argsort(lab, stable=True)
    lens = torch.bincount(lab, minlength=nlist).cpu().numpy()
    return X[order].cpu().numpy(), lens


def make_stream(a, themes, rng):
    """[(kind, agent, payload)] for every round."""
    sigma = 0.2 * np.sqrt(2.0) / np.sqrt(a.d)
    rounds = []
    for r in range(a.rounds):
        ops = []
        for s in range(1, a.agents + 1):
            ag = f"agent{s - 1}"
            th = themes[s]
            ins = (th[r % G] + sigma * rng.standard_normal((8, a.d))).astype(np.float32)
            ops.append(("insert", ag, ins))
            Q = np.empty((a.batch, a.d), dtype=np.float32)
            for j in range(a.batch):
                if rng.random() < a.explore:
                    v = rng.standard_normal(a.d)
                    Q[j] = (v / np.linalg.norm(v)).astype(np.float32)
                else:
                    Q[j] = (th[j % G] + sigma * rng.standard_normal(a.d)).astype(np.float32)
            ops.append(("search", ag, Q))
            ops.append(("end", ag, None))
        rounds.append(ops)
    return rounds


def run_stream(store, rounds, a, n_rounds, record_rounds, scalar_search):
    """Apply rounds to a Store; returns timing, level mix and the recorded
    search results of the first `record_rounds` rounds."""
    t_s = t_i = 0.0
    n_s = n_i = 0
    levels = {"L0": 0, "L1": 0, "L2": 0}
    early = 0
    rec = []
    for r in range(n_rounds):
        timed = r >= 1
        for kind, ag, payload in rounds[r]:
            if kind == "insert":
                t = time.perf_counter()
                store.insert(ag, ag, list(payload))
                dt = time.perf_counter() - t
                if timed:
                    t_i += dt
                    n_i += 1
            elif kind == "search":
                t = time.perf_counter()
                if scalar_search:
                    res = [store.search(ag, [ag, "static"], q, 10, a.nprobe) for q in payload]
                else:
                    res = store.search_batch(ag, [ag, "static"], payload, 10, a.nprobe)
                dt = time.perf_counter() - t
                if timed:
                    t_s += dt
                    n_s += len(payload)
                    for x in res:
                        levels[x.stats.level_reached] += 1
                        early += int(x.stats.early_terminated)
                if r < record_rounds:
                    rec.extend((list(x.ids), np.asarray(x.distances, np.float32).view(np.uint32).tolist(),
                                x.stats.level_reached, bool(x.stats.early_terminated),
                                int(x.stats.scanned_vectors)) for x in res)
            else:
                store.end_request(ag)
    ops = n_s + n_i
    return {"ms_per_op": 1000.0 * (t_s + t_i) / max(ops, 1),
            "search_ms_per_query": 1000.0 * t_s / max(n_s, 1),
            "insert8_ms": 1000.0 * t_i / max(n_i, 1),
            "searches_per_s": n_s / t_s if t_s else None,
            "levels": levels, "early_terminated": early, "timed_searches": n_s,
            "timed_insert_batches": n_i}, rec


def reference_modules():
    src = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(src, "agentmem")):
        src = "/root/reference/pkg/src"
    if not os.path.isdir(os.path.join(src, "agentmem")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="pk_numba_"))
    sys.path.insert(0, src)
    import agentmem

    return agentmem


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--agents", type=int, default=16)
    p.add_argument("--rows", type=int, default=250_000)
    p.add_argument("--d", type=int, default=1024)
    p.add_argument("--rounds", type=int, default=8)
    p.add_argument("--batch", type=int, default=32)
    p.add_argument("--nprobe", type=int, default=8)
    p.add_argument("--explore", type=float, default=0.25)
    p.add_argument("--alpha", type=float, nargs="*", default=[0.7, 0.0])
    p.add_argument("--ref-rounds", type=int, default=2, help="0: no reference arm")
    p.add_argument("--scalar", action="store_true", help="search() per query instead of search_batch")
    a = p.parse_args()

    import torch

    from paper_2602_21477_b200 import Store, StoreConfig
    from paper_2602_21477_b200 import _native as N
    from paper_2602_21477_b200.core import Metric
    from paper_2602_21477_b200.pnck import write_pnck

    N.load()
    dev = torch.device("cuda", 0)
    nlist = max(1, -(-a.rows // 2048))
    scopes = ["static"] + [f"agent{s}" for s in range(a.agents)]

    def scope_data(s):
        rows, lens = scope_rows(torch, dev, a.rows, a.d, nlist, 1000 + s)
        off = np.concatenate([[0], np.cumsum(lens)])
        ids = np.arange(s * a.rows, (s + 1) * a.rows, dtype=np.int64)
        return rows, [(ids[off[c]:off[c + 1]], rows[off[c]:off[c + 1]]) for c in range(nlist) if lens[c] > 0]

    rng = np.random.default_rng(7)
    themes = {}
    for s in range(1, a.agents + 1):
        pick = rng.choice(a.rows, G, replace=False)
        rows, _ = scope_rows(torch, dev, a.rows, a.d, nlist, 1000 + s)
        themes[s] = rows[np.sort(pick)].copy()
        del rows
    rounds = make_stream(a, themes, rng)
    out = {"workload": f"configs[2]: {a.agents} agents x {a.rows} x {a.d} (+ static {a.rows}), ~{nlist} "
                       f"lists per scope; per round and agent: insert 8 + search batch {a.batch} "
                       f"(k 10, nprobe {a.nprobe}, over [agent, static]; {int(100 * a.explore)}% exploration "
                       f"queries, the rest revisit the agent's 3 themes step-wise) + end_request; "
                       f"{a.rounds} rounds, round 0 untimed",
           "store_config": "defaults (cache, patterns, prefetch, profiles, hybrid graph ef 4, splits) "
                           "+ accelerator='none', threads=0",
           "modes": {}}
    recs = {}
    for alpha in a.alpha:
        t0 = time.perf_counter()
        store = Store(StoreConfig(dimension=a.d, alpha_et=alpha, accelerator="none", threads=0, seed=1))
        for s, sc in enumerate(scopes):
            if s:
                store.register_agent(sc)
            _, lists = scope_data(s)
            store.load_lists(sc, lists)
            del lists
        build_s = time.perf_counter() - t0
        timers = {}
        if os.environ.get("PK_TIME_CALLS"):  # garbage-collector pauses
            gc_t = [0.0]

            def gc_cb(phase, info, _t=[0.0]):
                if phase == "start":
                    _t[0] = time.perf_counter()
                else:
                    e = timers.setdefault(f"gc.gen{info['generation']}", [0, 0.0])
                    e[0] += 1
                    e[1] += time.perf_counter() - _t[0]
            gc.callbacks.append(gc_cb)
        if os.environ.get("PK_TIME_CALLS"):  # wall time per wrapped call (no profiler overhead)
            def wrap(obj, name, label):
                fn = getattr(obj, name)

                def timed(*args, **kw):
                    t = time.perf_counter()
                    try:
                        return fn(*args, **kw)
                    finally:
                        e = timers.setdefault(label, [0, 0.0])
                        e[0] += 1
                        e[1] += time.perf_counter() - t
                setattr(obj, name, timed)
            idx = store.index
            for m in ("agent_read", "agent_lists", "l1_place", "rows_put", "create_list", "graph_set", "append", "assign",
                      "flush"):
                if hasattr(idx, m):
                    wrap(idx, m, "index." + m)
            for m in ("_insert_impl", "_rows_for", "_materialize", "_search_read_phase", "_search_side_effects",
                      "_topk", "end_request", "_tick", "_state_key_for"):
                wrap(store, m, "store." + m)
            wrap(store.graph, "upload", "graph.upload")
            if os.environ.get("PK_TIME_CALLS") == "2":  # finer: the host policy's pieces (class level)
                from paper_2602_21477_b200 import cache as _c, fsm as _f, engine as _e
                for m in ("read_plan", "replay", "promote_and_capture", "_l1_decide", "_l1_place",
                          "_l1_capture", "threshold", "l1_listing_slots", "promote_to_l0"):
                    if hasattr(_c.MultiLevelCache, m):
                        wrap(_c.MultiLevelCache, m, "cache." + m)
                for m in ("match_and_predict", "match", "state_slots", "observe_completed"):
                    if hasattr(_f.PatternTable, m):
                        wrap(_f.PatternTable, m, "fsm." + m)
                for m in ("_hint_from", "_seq_D", "_cache_items", "_append_sequence", "_coarse_plan", "prefetch",
                          "_materialize"):
                    wrap(store, m, "store." + m)
                wrap(_e, "profile_order", "engine.profile_order")
            wrap(store.clusters, "create_cluster", "clusters.create_cluster")
        prof = None
        if os.environ.get("PK_PROFILE_OPS"):
            import cProfile

            prof = cProfile.Profile()
            prof.enable()
        res, rec = run_stream(store, rounds, a, a.rounds, a.ref_rounds, a.scalar)
        if prof is not None:
            import pstats

            prof.disable()
            st = pstats.Stats(prof, stream=sys.stderr)
            st.sort_stats("tottime").print_stats(30)
            st.sort_stats("cumulative").print_stats(50)
        if timers:
            res["call_ms"] = {k: {"calls": v[0], "total_ms": round(1e3 * v[1], 2),
                                  "ms_per_call": round(1e3 * v[1] / max(v[0], 1), 4)}
                              for k, v in sorted(timers.items(), key=lambda kv: -kv[1][1])}
        res["build_s"] = build_s
        res["clusters_after"] = len(store.clusters.clusters)
        out["modes"][f"alpha_et={alpha}"] = res
        recs[alpha] = rec
        print(json.dumps({f"alpha_et={alpha}": res}), file=sys.stderr, flush=True)
        store.close()
        del store
        gc.collect()
        torch.cuda.empty_cache()

    am = reference_modules() if a.ref_rounds > 0 else None
    if am is not None:
        ref = {}
        for alpha in a.alpha:
            t0 = time.perf_counter()
            rs = am.Store(am.StoreConfig(dimension=a.d, alpha_et=alpha, accelerator="none", threads=0, seed=1))
            with tempfile.TemporaryDirectory() as td:
                for s, sc in enumerate(scopes):
                    if s:
                        rs.register_agent(sc)
                    _, lists = scope_data(s)
                    path = os.path.join(td, "scope.pnck")
                    write_pnck(path, a.d, Metric.SQUARED_EUCLIDEAN,
                               [(np.zeros(a.d, np.float32), i, r) for i, r in lists])
                    del lists
                    rs.load_external_ivf(path, sc)
                    os.unlink(path)
            build_s = time.perf_counter() - t0
            res, rec = run_stream(rs, rounds, a, a.ref_rounds, a.ref_rounds, True)
            mine = recs[alpha]
            mism = {"ids": 0, "dist_bits": 0, "level": 0, "early": 0, "scanned": 0}
            for x, y in zip(mine, rec):
                mism["ids"] += x[0] != y[0]
                mism["dist_bits"] += x[1] != y[1]
                mism["level"] += x[2] != y[2]
                mism["early"] += x[3] != y[3]
                mism["scanned"] += x[4] != y[4]
            res.update(build_s=build_s, cores=1, compared_searches=len(rec), mismatches=mism,
                       sample=f"rounds 0..{a.ref_rounds - 1} of the same stream (round 0 untimed)")
            ref[f"alpha_et={alpha}"] = res
            print(json.dumps({f"reference alpha_et={alpha}": res}), file=sys.stderr, flush=True)
            del rs
            gc.collect()
        out["reference"] = ref
        for key, r in ref.items():
            mine = out["modes"][key]
            if r["ms_per_op"] and mine["ms_per_op"]:
                mine["speedup_vs_reference_ms_per_op"] = r["ms_per_op"] / mine["ms_per_op"]
    else:
        out["reference"] = "not run (--ref-rounds 0 or no baseline/_ref)"
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
