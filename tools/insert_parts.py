"""Wall time per piece of Store.insert (agent None, batch of 8, configs[4]
shape, no profiler): wrapped calls, microseconds per insert."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.getcwd())
from paper_2602_21477_b200 import Store, StoreConfig  # noqa: E402

d, nl, per = 768, 1024, 200
rng = np.random.default_rng(0)
base = rng.standard_normal((nl * per, d), dtype=np.float32)
base /= np.linalg.norm(base, axis=1, keepdims=True)
store = Store(StoreConfig(dimension=d, accelerator=os.environ.get("ACC", "simulated"), budget_bytes=1 << 28,
                          cache_enabled=False, splits_enabled=False))
store.load_lists("static", [(np.arange(i * per, (i + 1) * per, dtype=np.int64), base[i * per:(i + 1) * per])
                            for i in range(nl)])
vecs = rng.standard_normal((40000, d), dtype=np.float32)
vecs /= np.linalg.norm(vecs, axis=1, keepdims=True)
T = {}


def wrap(obj, name, label):
    fn = getattr(obj, name)

    def timed(*a, **k):
        t = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            e = T.setdefault(label, [0, 0.0])
            e[0] += 1
            e[1] += time.perf_counter() - t
    setattr(obj, name, timed)


for i in range(50):
    store.insert(None, "static", vecs[i * 8:(i + 1) * 8])
wrap(store, "_vectors", "store._vectors")
wrap(store, "_insert_run", "store._insert_run")
wrap(store, "_tick", "store._tick")
wrap(store.clusters, "assign_nearest_batch", "clusters.assign_nearest_batch")
wrap(store.clusters, "add_members_batch", "clusters.add_members_batch")
wrap(store.index, "append_rows", "index.append_rows")
wrap(store.index, "flush", "index.flush")
wrap(store.tier, "buffered_insert_batch", "tier.buffered_insert_batch")
N = 2000
t0 = time.perf_counter()
for i in range(50, 50 + N):
    store.insert(None, "static", vecs[i * 8:(i + 1) * 8])
store.index.flush()
tot = time.perf_counter() - t0
print(f"insert us/batch: {1e6 * tot / N:.1f}")
for k, (n, s) in sorted(T.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:32s} calls/insert {n / N:5.2f}  us/insert {1e6 * s / N:7.1f}")
