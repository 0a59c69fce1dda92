"""cProfile of Store.insert (agent None, batch of 8, configs[4] shape) --
where the host time of an insert goes."""
import cProfile
import os
import pstats
import sys

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
for i in range(50):
    store.insert(None, "static", list(vecs[i * 8:(i + 1) * 8]))
pr = cProfile.Profile()
pr.enable()
for i in range(50, 2050):
    store.insert(None, "static", list(vecs[i * 8:(i + 1) * 8]))
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(30)
