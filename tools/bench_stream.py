#!/usr/bin/env python3
"""configs[4]: insert-heavy streaming memory with the multi-level (HBM / pinned
host) tier, through the public Store API.

    python tools/bench_stream.py [--base 1000000] [--inserts 100000] [--budget-gb 1]

1M x 768 base (unit sphere, device k-means, nlist 1024) loaded into a
Store(accelerator="native", budget_bytes=1 GB of the 3.08 GB index): cold
lists live in pinned host memory, the hotset policy (ref/tiering.py:222-262)
runs every 64 operations.  The stream interleaves insert batches of 8
(agent=None: device assignment + in-place append, centroid maintenance every
256 member changes) with search batches of 256 queries (k 10, nprobe 32);
inserts and queries follow a Zipf(1.1) popularity over the clusters, the
locality an agent memory sees.  Prints one JSON line: insert vectors/s,
search QPS, tier residency and PCIe staging, and bit-exact parity of a query
sample against the C oracle over the final index.
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


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--base", type=int, default=1_000_000)
    p.add_argument("--d", type=int, default=768)
    p.add_argument("--nlist", type=int, default=1024)
    p.add_argument("--inserts", type=int, default=100_000)
    p.add_argument("--search-every", type=int, default=128, help="insert batches per search batch")
    p.add_argument("--budget-gb", type=float, default=1.0)
    p.add_argument("--zipf", type=float, default=1.1)
    p.add_argument("--parity", type=int, default=32)
    a = p.parse_args()

    import torch

    import bench as Bm
    from paper_2602_21477_b200 import Store, StoreConfig

    class A:  # build_shard arguments
        n, d, nlist, seed, kmeans_iters = a.base, a.d, a.nlist, 0, 2

    t0 = time.perf_counter()
    base, Xs, ids_sorted, lens, offs = Bm.build_shard(A, 0, torch.device("cuda", 0))
    rows_h = Xs.cpu().numpy()
    ids_h = ids_sorted.cpu().numpy()
    del Xs, ids_sorted
    torch.cuda.empty_cache()
    cfg = StoreConfig(dimension=a.d, accelerator="native", budget_bytes=int(a.budget_gb * (1 << 30)),
                      hotset_interval=64, cache_enabled=False, splits_enabled=False, seed=0)
    store = Store(cfg)
    lists = [(ids_h[offs[c]:offs[c] + lens[c]], rows_h[offs[c]:offs[c] + lens[c]])
             for c in range(a.nlist) if lens[c] > 0]
    store.load_lists("static", lists)
    build_s = time.perf_counter() - t0

    rng = np.random.default_rng(7)
    cids = sorted(store.clusters.clusters)
    cents = np.stack([store.clusters.clusters[c].centroid for c in cids])
    pop = 1.0 / np.arange(1, len(cids) + 1) ** a.zipf
    pop /= pop.sum()
    perm = rng.permutation(len(cids))

    def draw(n, sigma):
        c = perm[rng.choice(len(cids), size=n, p=pop)]
        x = cents[c] + sigma * rng.standard_normal((n, a.d), dtype=np.float32)
        return (x / np.linalg.norm(x, axis=1, keepdims=True)).astype(np.float32)

    nbatches = a.inserts // 8
    t_ins = t_srch = 0.0
    n_q = 0
    dev = torch.device("cuda", 0)
    staged0 = store.tier.metrics()["tier_staged_bytes_total"]
    for b in range(nbatches):
        vecs = draw(8, 0.05)
        t = time.perf_counter()
        store.insert(None, "static", list(vecs))
        t_ins += time.perf_counter() - t
        if (b + 1) % a.search_every == 0:
            Q = draw(256, 0.05)
            t = time.perf_counter()
            store.search_batch(None, ["static"], Q, 10, 32)
            torch.cuda.synchronize(dev)
            t_srch += time.perf_counter() - t
            n_q += 256
    m = store.tier.metrics()
    # parity: a query sample against the oracle over the final index
    from oracle import oracle as O

    Q = draw(a.parity, 0.05)
    res = store.search_batch(None, ["static"], Q, 10, 32)
    cl = store.clusters.clusters
    live = [c for c in sorted(cl) if cl[c].size > 0]
    flat = O.FlatIVF.from_lists([(cl[c].member_ids, cl[c].vectors) for c in live],
                                np.stack([cl[c].centroid for c in live]), np.array(live, np.int64))
    o_ids, o_d, o_n, _, _ = flat.search(Q, 32, 10, threads=os.cpu_count() or 1)
    mism = sum(int(r.ids != o_ids[i, :o_n[i]].tolist()) for i, r in enumerate(res))
    dmism = sum(int(np.asarray(r.distances, np.float32).view(np.uint32).tolist()
                    != o_d[i, :o_n[i]].view(np.uint32).tolist()) for i, r in enumerate(res))
    line = {
        "workload": f"configs[4]: {a.base} x {a.d} base (nlist {a.nlist}) + {nbatches * 8} inserts in "
                    f"batches of 8, one 256-query search batch per {a.search_every} insert batches, "
                    f"Zipf({a.zipf}) cluster popularity, native tier budget {a.budget_gb} GB",
        "insert_vectors_per_s": nbatches * 8 / t_ins,
        "insert_us_per_batch_of_8": 1e6 * t_ins / nbatches,
        "search_qps": n_q / t_srch if t_srch else None,
        "search_batches": n_q // 256,
        "tier": {k: v for k, v in m.items() if k.startswith("tier_") or k in ("residency_ratio", "resident_bytes")},
        "staged_gb_during_stream": (m["tier_staged_bytes_total"] - staged0) / 1e9,
        "pcie_gbs_effective": (m["tier_staged_bytes_total"] - staged0) / 1e9 / t_srch if t_srch else None,
        "parity_vs_oracle": {"queries": a.parity, "id_mismatch_queries": mism,
                             "dist_bit_mismatch_queries": dmism},
        "build_s": build_s,
    }
    print(json.dumps(line), flush=True)
    store.close()


if __name__ == "__main__":
    main()
