"""cProfile of the configs[4] insert stream (tools/bench_stream.py workload, inserts only)."""
import cProfile
import os
import pstats
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench as Bm
    from paper_2602_21477_b200 import Store, StoreConfig

    class A:
        n, d, nlist, seed, kmeans_iters = 1_000_000, 768, 1024, 0, 2

    base, Xs, ids_sorted, lens, offs = Bm.build_shard(A, 0, torch.device("cuda", 0))
    rows_h, ids_h = Xs.cpu().numpy(), ids_sorted.cpu().numpy()
    store = Store(StoreConfig(dimension=768, accelerator="native", budget_bytes=1 << 30, hotset_interval=64,
                              cache_enabled=False, splits_enabled=False, seed=0))
    store.load_lists("static", [(ids_h[offs[c]:offs[c] + lens[c]], rows_h[offs[c]:offs[c] + lens[c]])
                                for c in range(1024) if lens[c] > 0])
    rng = np.random.default_rng(7)
    cents = np.stack([store.clusters.clusters[c].centroid for c in sorted(store.clusters.clusters)])
    pop = 1.0 / np.arange(1, len(cents) + 1) ** 1.1
    pop /= pop.sum()
    vecs = cents[rng.choice(len(cents), 16000, p=pop)] + 0.05 * rng.standard_normal((16000, 768), dtype=np.float32)
    vecs /= np.linalg.norm(vecs, axis=1, keepdims=True)
    vecs = vecs.astype(np.float32)

    def run():
        for b in range(2000):
            store.insert(None, "static", list(vecs[b * 8:(b + 1) * 8]))

    cProfile.runctx("run()", globals(), locals(), "/tmp/stream.prof")
    pstats.Stats("/tmp/stream.prof").sort_stats("tottime").print_stats(22)


main()
