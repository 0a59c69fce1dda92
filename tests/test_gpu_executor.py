"""The executor plugin (SURVEY.md 8b layer 2): NativeAccelerator replays every
call the reference TierManager made on its SimulatedAccelerator
(tests/golden/make_golden.py --executor: buffered inserts, deletes, merged
searches, admissions / evictions / flushes, a failing allocation, failing
scans, resident splits).  Scans must return the same ids in the same order
and bit-identical distances; k-means must give the same labels, centres and
leave the store's random stream in the same state; `_mem` must hold the
uploaded snapshot; `allocated_bytes` must follow."""

import json

import numpy as np
import pytest

from replay import load_golden

pytestmark = pytest.mark.gpu


def test_executor_plugin_replays_reference_calls():
    from paper_2602_21477_b200.accelerator import NativeAccelerator
    from paper_2602_21477_b200.core import AcceleratorError, Metric

    g = load_golden("executor.npz")
    acc = NativeAccelerator(dimension=int(g["d"]))
    hmap = {}
    snap = {}  # reference-side contents per handle, to check _mem
    seen = {"scan": 0, "kmeans": 0, "alloc_fail": 0, "scan_fail": 0}
    for i in range(int(g["n"])):
        kind = str(g[f"{i}/kind"])
        if kind == "alloc":
            h = acc.alloc(int(g[f"{i}/nbytes"]))
            hmap[int(g[f"{i}/handle"])] = h
            snap[h] = (np.zeros((0, int(g["d"])), np.float32), np.zeros(0, np.int64))
        elif kind == "alloc_fail":
            acc.fail_next_alloc = True
            with pytest.raises(AcceleratorError):
                acc.alloc(int(g[f"{i}/nbytes"]))
            seen[kind] += 1
        elif kind == "upload":
            h = hmap[int(g[f"{i}/handle"])]
            mat, ids = g[f"{i}/mat"], g[f"{i}/ids"]
            acc.upload(h, mat, ids, bool(g[f"{i}/local"]))
            m0, i0 = snap[h]
            snap[h] = (np.concatenate([m0, mat.reshape(-1, m0.shape[1])]), np.concatenate([i0, ids]))
            got_m, got_i = acc._mem[h]
            assert np.array_equal(got_i, snap[h][1])
            assert np.array_equal(got_m.view(np.uint32), snap[h][0].view(np.uint32))
        elif kind == "release":
            h = hmap[int(g[f"{i}/handle"])]
            acc.release(h, int(g[f"{i}/nbytes"]))
            assert h not in acc._mem
        elif kind == "scan":
            h = hmap[int(g[f"{i}/handle"])]
            ids, d = acc.scan(h, g[f"{i}/q"], Metric.SQUARED_EUCLIDEAN)
            assert np.array_equal(ids, g[f"{i}/ids"])
            assert np.array_equal(np.asarray(d, np.float32).view(np.uint32),
                                  g[f"{i}/d"].astype(np.float32).view(np.uint32))
            seen[kind] += 1
        elif kind == "scan_fail":
            ref_h = int(g[f"{i}/handle"])
            if bool(g[f"{i}/injected"]):
                acc.fail_next_scan = True
            with pytest.raises(AcceleratorError):
                acc.scan(hmap.get(ref_h, -1), g[f"{i}/q"], Metric.SQUARED_EUCLIDEAN)
            seen[kind] += 1
        else:  # kmeans
            rng = np.random.default_rng()
            rng.bit_generator.state = json.loads(str(g[f"{i}/rng_before"]))
            labels, centers = acc.kmeans(g[f"{i}/mat"], int(g[f"{i}/k"]), rng, float(g[f"{i}/delta"]))
            assert np.array_equal(labels, g[f"{i}/labels"])
            assert np.array_equal(np.asarray(centers, np.float32).view(np.uint32),
                                  g[f"{i}/centers"].view(np.uint32))
            assert rng.bit_generator.state == json.loads(str(g[f"{i}/rng_after"]))
            seen[kind] += 1
    assert acc.allocated_bytes == int(g["allocated_bytes"])
    assert seen["scan"] > 20 and seen["kmeans"] >= 1 and seen["alloc_fail"] >= 1
    acc.close()
