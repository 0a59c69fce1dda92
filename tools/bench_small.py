"""Per-call latency of the small host-pointer entry points the agent path
uses: kernel-table distances (cache pools, L1 centroids), coarse_cids,
scan_lists and an 8-row append (us per call, median of 200)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_21477_b200 import DeviceIndex, kernels  # noqa: E402


def med_us(fn, reps=200):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return round(float(np.median(ts)) * 1e6, 1)


def main():
    rng = np.random.default_rng(0)
    d = 1024
    out = {}
    q = rng.normal(size=d).astype(np.float32)
    for n in (16, 64, 1024, 16384):
        m = rng.normal(size=(n, d)).astype(np.float32)
        out[f"sq_l2 n={n}"] = med_us(lambda: kernels.sq_l2(q, m))
    ix = DeviceIndex(d, 0, 0)
    for c in range(64):
        rows = rng.normal(size=(2000, d)).astype(np.float32)
        ix.create_list(c, 0, rows, np.arange(c * 2000, (c + 1) * 2000, dtype=np.int64))
    out["coarse_cids nprobe=8"] = med_us(lambda: ix.coarse_cids(q[None], [0], 8))
    cids = np.arange(8, dtype=np.int64)
    out["scan_lists 8 lists x 2000"] = med_us(lambda: ix.scan_lists(q, cids, 16000))
    nxt = [10**7]

    def app():
        ix.append(3, rng.normal(size=(8, d)).astype(np.float32), np.arange(nxt[0], nxt[0] + 8))
        nxt[0] += 8
        ix.flush()

    out["append 8 rows"] = med_us(app, 100)
    ix.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
