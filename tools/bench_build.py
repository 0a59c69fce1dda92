#!/usr/bin/env python3
"""Store.bulk_build through the public API:
k-means++ seeding, <=10 Lloyd iterations and the cluster creation with the
matrix resident in HBM.  configs[0] (100K x 384, split_target 391 -> 256
lists; the reference needs 94-128 s on one CPU core) and configs[1]
(1M x 768, split_target 2048 -> 489 lists; infeasible on the reference CPU
path).  One JSON line per case."""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2602_21477_b200 import Store, StoreConfig

    for name, n, d, target in (("configs[0]", 100_000, 384, 391), ("configs[1]", 1_000_000, 768, 2048)):
        rng = np.random.default_rng(np.random.PCG64(0))
        x = rng.standard_normal((n, d), dtype=np.float32)
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        store = Store(StoreConfig(dimension=d, seed=0, split_target=target, split_threshold=1 << 30,
                                  cache_enabled=False, splits_enabled=False, accelerator="none"))
        t0 = time.perf_counter()
        ids = store.bulk_build("static", x)
        dt = time.perf_counter() - t0
        sizes = [c.size for c in store.clusters.clusters.values()]
        print(json.dumps({"case": name, "n": n, "d": d, "lists": len(sizes), "bulk_build_s": dt,
                          "rows_per_s": n / dt, "min_list": int(min(sizes)), "max_list": int(max(sizes)),
                          "ids": len(ids)}), flush=True)
        store.close()


if __name__ == "__main__":
    main()
