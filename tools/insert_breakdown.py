"""Where an insert batch of 8 spends its time (configs[4] shape, 1024 lists,
d 768): device assignment alone, the append flush alone, the whole
Store.insert, and the Store.insert loop without the flush."""
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
acc = os.environ.get("ACC", "simulated")
store = Store(StoreConfig(dimension=d, accelerator=acc, budget_bytes=1 << 28, cache_enabled=False,
                          splits_enabled=False))
store.load_lists("static", [(np.arange(i * per, (i + 1) * per, dtype=np.int64), base[i * per:(i + 1) * per])
                            for i in range(nl)])
vecs = rng.standard_normal((40000, d), dtype=np.float32)
vecs /= np.linalg.norm(vecs, axis=1, keepdims=True)
ix = store.index
R = 1000


def timeit(f, n=R):
    f(0)
    t = time.perf_counter()
    for i in range(1, n + 1):
        f(i)
    return (time.perf_counter() - t) / n * 1e6


out = {}
out["assign_us"] = timeit(lambda i: ix.assign(vecs[i * 8:(i + 1) * 8], 0))
cids = np.arange(8) * 100


def app(i):
    for j in range(8):
        ix.append(int(cids[j]), vecs[i * 8 + j:i * 8 + j + 1], np.array([10**7 + i * 8 + j]))
    ix.flush()


out["append8_flush_us"] = timeit(app, 200)
k0 = 2000


def ins(i):
    store.insert(None, "static", list(vecs[(k0 + i) * 8:(k0 + i + 1) * 8]))


out["store_insert_us"] = timeit(ins)
out["store_insert_plus_flush_us"] = timeit(lambda i: (ins(i + R + 5), ix.flush()))
out["accelerator"] = acc
print(out)
