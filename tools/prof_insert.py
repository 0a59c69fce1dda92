"""Insert latency (configs[4] shape): batches of 8 through Store.insert on a
1024-list 768-d index, native tier.  Prints us per batch (appends flushed by
the next batch / at the end), then a cProfile of the same loop."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, os.getcwd())
from paper_2602_21477_b200 import Store, StoreConfig  # noqa: E402

d, nl, per = 768, 1024, 200
rng = np.random.default_rng(0)
base = rng.standard_normal((nl * per, d), dtype=np.float32)
base /= np.linalg.norm(base, axis=1, keepdims=True)
store = Store(StoreConfig(dimension=d, accelerator=os.environ.get("ACC", "native"), budget_bytes=1 << 28,
                          cache_enabled=False, splits_enabled=False))
lists = [(np.arange(i * per, (i + 1) * per, dtype=np.int64), base[i * per:(i + 1) * per]) for i in range(nl)]
store.load_lists("static", lists)
vecs = rng.standard_normal((16000, d), dtype=np.float32)
vecs /= np.linalg.norm(vecs, axis=1, keepdims=True)


def run(lo, hi):
    for b in range(lo, hi):
        store.insert(None, "static", list(vecs[b * 8:(b + 1) * 8]))
    store.index.flush()


run(0, 50)
t = time.perf_counter()
run(50, 1050)
print("us per batch of 8:", (time.perf_counter() - t) * 1e3)
cProfile.run("run(1050, 1550)", "/tmp/ins.prof")
pstats.Stats("/tmp/ins.prof").sort_stats("tottime").print_stats(18)
