"""Sharded search host logic on CPU: placement, block
layout (against the C-ABI), and the world_size-2 gloo path -- placement,
centroid replication, block all-gather and merge -- whose merged answer must
equal the single-index oracle bit for bit."""

import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from paper_2602_21477_b200 import _native
from paper_2602_21477_b200 import build as B
from paper_2602_21477_b200.sharded import block_offsets, place_lists


def test_place_lists_balanced_and_deterministic():
    rng = np.random.default_rng(0)
    sizes = rng.integers(1, 2000, size=1000)
    for world in (1, 2, 4, 8):
        o1 = place_lists(sizes, world)
        o2 = place_lists(sizes.copy(), world)
        assert np.array_equal(o1, o2)
        assert set(o1.tolist()) <= set(range(world))
        load = np.bincount(o1, weights=sizes, minlength=world)
        assert load.max() - load.min() <= sizes.max()  # greedy LPT bound
    assert place_lists([], 4).shape == (0,)
    # ties: equal sizes go round-robin from rank 0
    assert place_lists([5, 5, 5, 5], 2).tolist() == [0, 1, 0, 1]


def test_block_layout_matches_library():
    B.build()
    lib = _native.load()
    for Bq, kk in ((1, 1), (3, 10), (256, 10), (255, 64), (0, 5)):
        assert lib.pk_shard_block_bytes(Bq, kk) == block_offsets(Bq, kk)["total"]
        o = block_offsets(Bq, kk)
        assert o["n"] + 4 * Bq <= o["total"]
        assert o["dists"] % 8 == 0 and o["scanned"] % 8 == 0


def _make_lists(seed, nlist, d):
    rng = np.random.default_rng(seed)
    cents = rng.normal(size=(nlist, d)).astype(np.float32)
    lists, nid = [], 0
    for c in range(nlist):
        n = int(rng.integers(0, 60)) if c % 7 else 0  # some empty lists
        n = max(n, 1) if c % 11 == 0 else n
        rows = (cents[c] + 0.4 * rng.normal(size=(n, d))).astype(np.float32)
        ids = rng.permutation(np.arange(nid, nid + n)).astype(np.int64)
        nid += n
        lists.append((ids, rows))
    keep = [c for c in range(nlist) if len(lists[c][0]) > 0]
    Q = (cents[rng.integers(0, nlist, 24)] + 0.4 * rng.normal(size=(24, d))).astype(np.float32)
    # exact duplicate rows across two lists -> equal distances, ties by id
    if len(keep) >= 2:
        a, b = keep[0], keep[1]
        lists[b] = (lists[b][0], np.concatenate([lists[a][1][:1], lists[b][1][1:]]))
    return [lists[c] for c in keep], [100 + 3 * c for c in keep], Q


INS_INTERVAL = 5  # small, so maintenance fires many times inside one batch


def _insert_batch(seed, d):
    rng = np.random.default_rng(seed + 100)
    X = (0.8 * rng.normal(size=(120, d))).astype(np.float32)
    return X, np.arange(10**6, 10**6 + len(X), dtype=np.int64)


def _sequential_inserts(lists, cids, X, ids, interval):
    """The reference's per-vector insert (ref/engine.py:647-660): assign to the
    nearest list, append, recompute the centroid when its dirty count
    reaches the interval."""
    lists = [(i.copy(), r.copy()) for i, r in lists]
    cents = [O.centroid(r) for _, r in lists]
    dirty = [0] * len(lists)
    cid_arr = np.array(cids, np.int64)
    assigned = []
    for x, iid in zip(X, ids):
        c = O.assign_nearest(x, np.stack(cents), cid_arr)
        j = cids.index(c)
        assigned.append(c)
        lists[j] = (np.append(lists[j][0], iid), np.concatenate([lists[j][1], x[None]]))
        dirty[j] += 1
        if dirty[j] >= interval:
            cents[j] = O.centroid(lists[j][1])
            dirty[j] = 0
    return lists, np.stack(cents), np.array(assigned, np.int64)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, seed, nprobe, kk):
    import torch.distributed as dist

    from paper_2602_21477_b200.sharded import ShardedIndex
    from shard_oracle import OracleShard

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    d = 24
    lists, cids, Q = _make_lists(seed, 40, d)
    sh = ShardedIndex(d, local=OracleShard(d))
    owners = sh.load(cids, [0] * len(cids), [len(i) for i, _ in lists], lambda i: lists[i][::-1])
    out = sh.search(Q, [0], nprobe, kk)
    # dispatch/combine: each rank brings its own slice of the queries
    per = len(Q) // world
    mine = Q[rank * per:(rank + 1) * per]
    dsp = sh.search_dispatch(mine, [0], nprobe, kk)
    # inserts (every rank the same batch): assignment over replicated centroids,
    # owner appends, maintenance recompute broadcast from the owner
    Xi, ids_i = _insert_batch(seed, d)
    assigned = sh.insert(Xi, ids_i, 0, maintenance_interval=INS_INTERVAL)
    ins = sh.search(Q, [0], nprobe, kk)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), ids=out.ids, d=out.dists, cids=out.cids,
             n=out.counts, sc=out.scanned, owners=owners, dids=dsp.ids, dd=dsp.dists,
             dc=dsp.cids, dn=dsp.counts, dsc=dsp.scanned, assigned=assigned, iids=ins.ids,
             idd=ins.dists, icids=ins.cids, in_=ins.counts, isc=ins.scanned)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_search_equals_single_index(tmp_path, world):
    import torch.multiprocessing as mp

    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    seed, nprobe, kk = 3, 9, 10
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), seed, nprobe, kk), nprocs=world,
             join=True)
    d = 24
    lists, cids, Q = _make_lists(seed, 40, d)
    cents = np.stack([O.centroid(r) for _, r in lists])
    flat = O.FlatIVF.from_lists(lists, cents, np.array(cids, np.int64))
    ids, dd, cnt, _, sc = flat.search(Q, nprobe, kk)
    id2cid = {int(i): c for (ii, _), c in zip(lists, cids) for i in ii}
    res = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    for r in res:
        assert np.array_equal(r["ids"], ids)
        assert np.array_equal(r["d"].view(np.uint32), dd.view(np.uint32))
        assert np.array_equal(r["n"], cnt)
        assert np.array_equal(r["sc"], sc)
        exp_c = np.vectorize(lambda i: id2cid.get(int(i), -1), otypes=[np.int64])(ids)
        assert np.array_equal(r["cids"], exp_c)
    # dispatch/combine: rank r answered its own slice of the queries
    per = len(Q) // world
    for r, x in enumerate(res):
        sl = slice(r * per, (r + 1) * per)
        assert np.array_equal(x["dids"], ids[sl])
        assert np.array_equal(x["dd"].view(np.uint32), dd[sl].view(np.uint32))
        assert np.array_equal(x["dn"], cnt[sl])
        assert np.array_equal(x["dsc"], sc[sl])
        assert np.array_equal(x["dc"], exp_c[sl])
    # inserts: same assignment as the sequential reference path, and the
    # search after them equals the single index built by that path
    Xi, ids_i = _insert_batch(seed, d)
    lists2, cents2, assigned = _sequential_inserts(lists, cids, Xi, ids_i, INS_INTERVAL)
    flat2 = O.FlatIVF.from_lists(lists2, cents2, np.array(cids, np.int64))
    ids2, dd2, cnt2, _, sc2 = flat2.search(Q, nprobe, kk)
    id2cid2 = {int(i): c for (ii, _), c in zip(lists2, cids) for i in ii}
    for r in res:
        assert np.array_equal(r["assigned"], assigned)
        assert np.array_equal(r["iids"], ids2)
        assert np.array_equal(r["idd"].view(np.uint32), dd2.view(np.uint32))
        assert np.array_equal(r["in_"], cnt2)
        assert np.array_equal(r["isc"], sc2)
        assert np.array_equal(r["icids"], np.vectorize(lambda i: id2cid2.get(int(i), -1),
                                                       otypes=[np.int64])(ids2))
    assert not np.array_equal(cents2, np.stack([O.centroid(r) for _, r in lists]))
    # every rank derived the same placement, and both ranks own lists
    assert np.array_equal(res[0]["owners"], res[1]["owners"])
    assert set(res[0]["owners"].tolist()) == {0, 1}
