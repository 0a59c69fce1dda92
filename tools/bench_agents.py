#!/usr/bin/env python3
"""configs[2]: many agents with per-agent scopes and the multi-level cache,
mixed insert / search stream, through the public Store API.

    python tools/bench_agents.py [--agents 16] [--rows 250000] [--d 1024] [--rounds 20]

Each agent owns a scope of `rows` unit-sphere vectors (a themed mixture: 8
centres per agent, sigma = 0.2 sqrt(2)/sqrt(d) like bench/workload.py:73-76)
built into an IVF by device k-means (~2033 rows per list, the default
split_target) and loaded with load_lists; the static scope has `rows`
vectors too.  A round gives every agent one insert batch of 8 (staged into
its cache, merged down as clusters when an L1 pool fills) and 4 searches
(k 10, nprobe 8) over [agent, static] near its current theme, ending a
request every 8 ops.  Reports ms per op, searches/s and the cache-level /
early-termination mix for alpha_et 0.7 (cache on) and alpha_et 0.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build_scope(torch, N, n, d, nlist, seed, dev, centres):
    """Themed rows around `centres` + device k-means (kmeans_assign arithmetic)."""
    g = torch.Generator(device=dev).manual_seed(seed)
    sigma = 0.2 * np.sqrt(2.0) / np.sqrt(d)
    C = torch.from_numpy(centres).to(dev)
    pick = torch.randint(0, len(centres), (n,), generator=g, device=dev)
    X = C[pick] + sigma * torch.randn(n, d, generator=g, device=dev)
    X = (X / X.norm(dim=1, keepdim=True)).float().contiguous()
    cents = X[torch.randperm(n, generator=g, device=dev)[:nlist]].contiguous()
    labels = torch.empty(n, dtype=torch.int64, device=dev)
    dists = torch.empty(n, dtype=torch.float64, device=dev)
    for _ in range(2):
        torch.cuda.synchronize()
        N.check(N.lib().pk_kmeans_assign(X.data_ptr(), n, cents.data_ptr(), nlist, d, labels.data_ptr(),
                                         dists.data_ptr(), N.PK_DEVICE_PTRS))
        sums = torch.zeros(nlist, d, dtype=torch.float64, device=dev)
        sums.index_add_(0, labels, X.double())
        cnt = torch.bincount(labels, minlength=nlist).clamp(min=1).double()
        cents = (sums / cnt[:, None]).float().contiguous()
    order = torch.argsort(labels, stable=True)
    rows = X[order].cpu().numpy()
    lens = torch.bincount(labels, minlength=nlist).cpu().numpy()
    return rows, order.cpu().numpy(), lens


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--agents", type=int, default=16)
    p.add_argument("--rows", type=int, default=250_000)
    p.add_argument("--d", type=int, default=1024)
    p.add_argument("--rounds", type=int, default=20)
    p.add_argument("--nprobe", type=int, default=8)
    a = p.parse_args()

    import torch

    from paper_2602_21477_b200 import Store, StoreConfig
    from paper_2602_21477_b200 import _native as N

    N.load()
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(5)
    nlist = max(1, -(-a.rows // 2048))
    out = {"workload": f"configs[2]: {a.agents} agents x {a.rows} x {a.d} (+ static {a.rows}), "
                       f"nlist {nlist} per scope, rounds of insert-8 + 4 searches per agent "
                       f"(k 10, nprobe {a.nprobe}) over [agent, static]", "modes": {}}
    themes = {}
    for alpha in (0.7, 0.0):
        t0 = time.perf_counter()
        store = Store(StoreConfig(dimension=a.d, alpha_et=alpha, cache_enabled=True,
                                  accelerator="none", splits_enabled=False,
                                  ef_search_factor=1 << 20, seed=1))
        nid = 0
        for s in range(a.agents + 1):
            scope = "static" if s == 0 else store.register_agent(f"agent{s - 1}")
            centres = rng.standard_normal((8, a.d)).astype(np.float32) if s not in themes else themes[s]
            centres /= np.linalg.norm(centres, axis=1, keepdims=True)
            themes[s] = centres
            rows, order, lens = build_scope(torch, N, a.rows, a.d, nlist, 100 + s, dev, centres)
            ids = (order + nid).astype(np.int64)
            nid += a.rows
            off = np.concatenate([[0], np.cumsum(lens)])
            store.load_lists(scope, [(ids[off[c]:off[c + 1]], rows[off[c]:off[c + 1]])
                                     for c in range(nlist) if lens[c] > 0])
        build_s = time.perf_counter() - t0
        sigma = 0.2 * np.sqrt(2.0) / np.sqrt(a.d)
        for s in range(1, a.agents + 1):  # untimed warm-up op per agent (first-call costs)
            ag = f"agent{s - 1}"
            store.search(ag, [ag, "static"], themes[s][7], 10, a.nprobe)
        n_s = n_i = 0
        levels = {"L0": 0, "L1": 0, "L2": 0}
        early = 0
        t_s = t_i = 0.0
        prof = None
        if os.environ.get("PK_PROFILE_OPS") and alpha == 0.7:  # cProfile of the op loop only
            import cProfile

            prof = cProfile.Profile()
            prof.enable()
        for r in range(a.rounds):
            for s in range(1, a.agents + 1):
                ag = f"agent{s - 1}"
                centre = themes[s][(r // 2) % 8]
                vecs = (centre + sigma * rng.standard_normal((8, a.d))).astype(np.float32)
                t = time.perf_counter()
                store.insert(ag, ag, list(vecs))
                t_i += time.perf_counter() - t
                n_i += 1
                for _ in range(4):
                    q = (centre + sigma * rng.standard_normal(a.d)).astype(np.float32)
                    t = time.perf_counter()
                    res = store.search(ag, [ag, "static"], q, 10, a.nprobe)
                    t_s += time.perf_counter() - t
                    n_s += 1
                    levels[res.stats.level_reached] += 1
                    early += int(res.stats.early_terminated)
                if r % 2 == 1:
                    store.end_request(ag)
        if prof is not None:
            import pstats

            prof.disable()
            st = pstats.Stats(prof, stream=sys.stderr)
            st.sort_stats("tottime").print_stats(30)
            st.sort_stats("cumulative").print_stats(40)
        out["modes"][f"alpha_et={alpha}"] = {
            "ms_per_op": 1000.0 * (t_s + t_i) / (n_s + n_i),
            "search_ms": 1000.0 * t_s / n_s, "insert8_ms": 1000.0 * t_i / n_i,
            "searches_per_s": n_s / t_s, "levels": levels, "early_terminated": early,
            "searches": n_s, "insert_batches": n_i, "build_s": build_s,
            "clusters": len(store.clusters.clusters)}
        store.close()
        del store
        torch.cuda.empty_cache()
    out["reference_cpu_ms_per_op"] = "22.6 (SURVEY.md 8f, 16 agents d=1024, same op mix, 1 core)"
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
