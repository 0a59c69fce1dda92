#!/usr/bin/env python3
"""PNCK exchange at configs[1] scale: export_ivf of a 1M x 768
store and load_external_ivf into a fresh store (the reference takes ~29 s per
1M x 768 load with a per-vector loop, ref/persist.py:397-424)."""

import json
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2602_21477_b200 import Store, StoreConfig

    n, d, nl = 1_000_000, 768, 1024
    rng = np.random.default_rng(1)
    x = rng.standard_normal((n, d), dtype=np.float32)
    lab = rng.integers(0, nl, n)
    order = np.argsort(lab, kind="stable")
    bounds = np.concatenate([[0], np.cumsum(np.bincount(lab, minlength=nl))])
    cfg = dict(dimension=d, cache_enabled=False, splits_enabled=False, accelerator="none")
    a = Store(StoreConfig(**cfg))
    a.load_lists("static", [(order[bounds[c]:bounds[c + 1]].astype(np.int64), x[order[bounds[c]:bounds[c + 1]]])
                            for c in range(nl)])
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "x.pnck")
        t0 = time.perf_counter()
        a.export_ivf(path)
        t_exp = time.perf_counter() - t0
        b = Store(StoreConfig(**cfg))
        t0 = time.perf_counter()
        cnt = b.load_external_ivf(path, "static")
        t_load = time.perf_counter() - t0
        size = os.path.getsize(path)
    q = x[:64] + 0.01
    ra = a.search_batch(None, ["static"], q, 10, 16)
    rb = b.search_batch(None, ["static"], q, 10, 16)
    same = all(u.ids == v.ids and u.distances == v.distances for u, v in zip(ra, rb))
    print(json.dumps({"rows": n, "d": d, "lists": cnt, "file_gb": size / 1e9, "export_s": t_exp,
                      "load_s": t_load, "roundtrip_results_identical": same}), flush=True)


if __name__ == "__main__":
    main()
