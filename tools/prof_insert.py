import cProfile, pstats, sys, os, numpy as np, time
sys.path.insert(0, os.getcwd())
from paper_2602_21477_b200 import Store, StoreConfig
d=768
rng=np.random.default_rng(0)
base=rng.standard_normal((100000,d),dtype=np.float32); base/=np.linalg.norm(base,axis=1,keepdims=True)
store=Store(StoreConfig(dimension=d, accelerator="native", budget_bytes=1<<28, cache_enabled=False, splits_enabled=False))
lists=[(np.arange(i*1000,(i+1)*1000,dtype=np.int64), base[i*1000:(i+1)*1000]) for i in range(100)]
store.load_lists("static", lists)
vecs=rng.standard_normal((8000,d),dtype=np.float32); vecs/=np.linalg.norm(vecs,axis=1,keepdims=True)
def run():
    for b in range(1000):
        store.insert(None,"static",list(vecs[b*8:(b+1)*8]))
    store.index.flush()
t=time.perf_counter(); run(); print("us/batch", (time.perf_counter()-t)*1e3)
cProfile.run("run()", "/tmp/ins.prof")
p=pstats.Stats("/tmp/ins.prof"); p.sort_stats("cumulative").print_stats(25)
