#!/usr/bin/env python3
"""configs[4]: insert-heavy streaming memory with the multi-level (HBM / pinned
host) tier, through the public Store API, beside the reference's own tiered
path on the same host.

    python tools/bench_stream.py [--base 1000000] [--inserts 500000] [--budget-gb 1]
                                 [--ref-inserts 2000] [--ref-queries 16]

1M x 768 base (bench.py's index: seeded device rows, nlist 1024 nearest-seed
partition) loaded into a Store(accelerator="native", budget_bytes=1 GB of the
3.08 GB index): cold lists live in pinned host memory, the hotset policy
(ref/tiering.py:222-262) runs every 64 operations.  The stream: 500K inserts
in batches of 8 (agent=None: device assignment + in-place append, centroid
maintenance every 256 member changes, ref/engine.py:571-605, 647-660) with a
256-query search batch (k 10, nprobe 32) every 128 insert batches; inserts and
queries follow a Zipf(1.1) popularity over the clusters.

The reference arm: the reference package's Store (baseline/_ref) with
accelerator="simulated" at the same budget_bytes (ref/tiering.py:85-147,
280-290), the same base loaded through its load_external_ivf, the same first
``--ref-inserts`` inserts and a ``--ref-queries`` search sample -- its CPU
rates on this host, and its answers compared with ours at the same point of
the stream (exhaustive-ef reference config: identical results
expected).  Prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def reference_store(d, budget, nlist, nprobe, pnck_path):
    """The reference Store (its own package, baseline/_ref) on the same base."""
    src = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(src, "agentmem")):
        src = "/root/reference/pkg/src"
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="pk_numba_"))
    sys.path.insert(0, src)
    from agentmem import Store as RStore
    from agentmem import StoreConfig as RConfig

    cfg = RConfig(dimension=d, accelerator="simulated", budget_bytes=budget, hotset_interval=64,
                  cache_enabled=False, splits_enabled=False, seed=0,
                  ef_search_factor=max(4, -(-nlist // nprobe) * 2))
    st = RStore(cfg)
    t = time.perf_counter()
    st.load_external_ivf(pnck_path, "static")
    return st, time.perf_counter() - t


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--base", type=int, default=1_000_000)
    p.add_argument("--d", type=int, default=768)
    p.add_argument("--nlist", type=int, default=1024)
    p.add_argument("--inserts", type=int, default=500_000)
    p.add_argument("--search-every", type=int, default=128, help="insert batches per search batch")
    p.add_argument("--budget-gb", type=float, default=1.0)
    p.add_argument("--zipf", type=float, default=1.1)
    p.add_argument("--parity", type=int, default=32)
    p.add_argument("--ref-inserts", type=int, default=2000, help="0: no reference arm")
    p.add_argument("--ref-queries", type=int, default=16)
    a = p.parse_args()

    import torch

    import bench as Bm
    from paper_2602_21477_b200 import Store, StoreConfig
    from paper_2602_21477_b200.core import Metric
    from paper_2602_21477_b200.pnck import write_pnck

    t0 = time.perf_counter()
    dev = torch.device("cuda", 0)
    ba = Bm.resolve(argparse.Namespace(config="1", mode="auto", n=a.base, d=a.d, nlist=a.nlist,
                                       nprobe=32, k=10, batch=256, seed=0), 1)
    X, order, lens, offs = Bm.build_partition(ba, dev)
    rows_h = np.empty((a.base, a.d), dtype=np.float32)
    for i in range(0, a.base, 1 << 20):
        rows_h[i:i + (1 << 20)] = X[order[i:i + (1 << 20)]].cpu().numpy()
    ids_h = order.cpu().numpy().astype(np.int64)
    del X, order
    torch.cuda.empty_cache()
    budget = int(a.budget_gb * (1 << 30))
    # the same coarse ef as the reference arm (exhaustive: the flat oracle
    # over the final index applies, and both stores probe the same lists)
    cfg = StoreConfig(dimension=a.d, accelerator="native", budget_bytes=budget, hotset_interval=64,
                      cache_enabled=False, splits_enabled=False, seed=0,
                      ef_search_factor=max(4, -(-a.nlist // 32) * 2))
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
    ref_batches = min(a.ref_inserts // 8, nbatches)
    stream = [draw(8, 0.05) for _ in range(ref_batches)]  # the prefix both arms run
    Qref = draw(max(a.ref_queries, 1), 0.05)

    # ---- reference arm: same base, same first inserts, same query sample
    ref = None
    if ref_batches:
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "base.pnck")
            write_pnck(path, a.d, Metric.SQUARED_EUCLIDEAN,
                       [(np.zeros(a.d, np.float32), i, r) for i, r in lists])
            rst, load_s = reference_store(a.d, budget, a.nlist, 32, path)
        t = time.perf_counter()
        for v in stream:
            rst.insert(None, "static", list(v))
        r_ins = time.perf_counter() - t
        t = time.perf_counter()
        r_res = [rst.search(None, ["static"], q, 10, 32) for q in Qref]
        r_srch = time.perf_counter() - t
        ref = {"insert_vectors_per_s": ref_batches * 8 / r_ins,
               "insert_us_per_batch_of_8": 1e6 * r_ins / ref_batches,
               "search_qps": len(Qref) / r_srch, "cores": 1,
               "sample": f"first {ref_batches * 8} inserts of the stream, {len(Qref)} queries after them",
               "load_external_ivf_s": load_s,
               "config": "reference agentmem Store, accelerator='simulated', same budget_bytes, "
                         "cache off, splits off, exhaustive ef (ef_search_factor "
                         f"{rst.cfg.ef_search_factor})",
               "tier_metrics": {k: v for k, v in rst.tier.metrics().items()
                                if k in ("residency_ratio", "buffer_flush_count", "resident_bytes")}}

    # ---- our stream (the reference's prefix first: compare at that point)
    t_ins = t_srch = 0.0
    n_q = 0
    staged0 = store.tier.metrics()["tier_staged_bytes_total"]
    same = None
    T = {}
    if os.environ.get("PK_TIME_CALLS"):  # wall time per wrapped call (no profiler overhead)
        def wrap(obj, name, label):
            fn = getattr(obj, name)

            def timed(*a_, **k_):
                t_ = time.perf_counter()
                try:
                    return fn(*a_, **k_)
                finally:
                    e = T.setdefault(label, [0, 0.0])
                    e[0] += 1
                    e[1] += time.perf_counter() - t_
            setattr(obj, name, timed)
        for m in ("_vectors", "_insert_run", "_tick"):
            wrap(store, m, "store." + m)
        wrap(store.clusters, "assign_nearest_batch", "clusters.assign_nearest_batch")
        wrap(store.clusters, "add_members_batch", "clusters.add_members_batch")
        wrap(store.index, "flush", "index.flush")
        wrap(store.index, "set_resident", "index.set_resident")
        wrap(store.tier, "hotset_update", "tier.hotset_update")
        wrap(store.tier, "buffered_insert_batch", "tier.buffered_insert_batch")
    prof = None
    if os.environ.get("PK_PROFILE_STREAM"):  # cProfile of the insert path (batches 2000..)
        import cProfile

        prof = cProfile.Profile()
    for b in range(nbatches):
        if prof is not None and b == min(2000, nbatches // 2):
            prof.enable()
        vecs = stream[b] if b < ref_batches else draw(8, 0.05)
        t = time.perf_counter()
        store.insert(None, "static", list(vecs))
        t_ins += time.perf_counter() - t
        if ref is not None and b == ref_batches - 1:
            ours = store.search_batch(None, ["static"], Qref, 10, 32)
            same = {"queries": len(Qref),
                    "id_mismatch_queries": sum(int(o.ids != r.ids) for o, r in zip(ours, r_res)),
                    "dist_bit_mismatch_queries": sum(
                        int(np.asarray(o.distances, np.float32).view(np.uint32).tolist()
                            != np.asarray(r.distances, np.float32).view(np.uint32).tolist())
                        for o, r in zip(ours, r_res))}
        if (b + 1) % a.search_every == 0:
            Q = draw(256, 0.05)
            t = time.perf_counter()
            store.search_batch(None, ["static"], Q, 10, 32)
            torch.cuda.synchronize(dev)
            t_srch += time.perf_counter() - t
            n_q += 256
    if prof is not None:
        import pstats

        prof.disable()
        pstats.Stats(prof, stream=sys.stderr).sort_stats("tottime").print_stats(30)
    if T:
        for k, (n_, s_) in sorted(T.items(), key=lambda kv: -kv[1][1]):
            print(f"  {k:32s} calls/batch {n_ / nbatches:6.3f}  us/batch {1e6 * s_ / nbatches:8.1f}",
                  file=sys.stderr)
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
        "reference_simulated_tier": ref,
        "same_answers_as_reference_at_its_sample": same,
        "build_s": build_s,
    }
    print(json.dumps(line), flush=True)
    store.close()


if __name__ == "__main__":
    main()
