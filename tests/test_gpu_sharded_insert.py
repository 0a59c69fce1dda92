"""Sharded inserts on the device, two PROCESSES over a
gloo group, both ranks on cuda:0 of this one-GPU box: every rank assigns the
same batch over the replicated centroids, owners append, maintenance
recomputes are broadcast from the owner.  The assignment and the search
after the inserts must equal the reference's sequential insert path
(restated with the C oracle) bit for bit."""

import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from oracle import oracle as O  # noqa: E402
from test_sharded import _sequential_inserts  # noqa: E402

D, NLIST, NPROBE, KK, INTERVAL = 64, 24, 5, 10, 9


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data():
    from test_gpu_sharded import _lists

    lists, Q = _lists(4242, NLIST, D, 300)
    rng = np.random.default_rng(5)
    X = (rng.normal(size=(400, D))).astype(np.float32)
    return lists, Q, X, np.arange(5 * 10**6, 5 * 10**6 + len(X), dtype=np.int64)


def _worker(rank, world, port, outdir):
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch
    import torch.distributed as dist

    from paper_2602_21477_b200.sharded import ShardedIndex

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    lists, Q, X, ids = _data()
    cids = list(range(NLIST))
    sh = ShardedIndex(D, 0, 0)
    owners = sh.load(cids, [0] * NLIST, [len(i) for i, _ in lists], lambda i: lists[i][::-1])
    assigned = sh.insert(X, ids, 0, maintenance_interval=INTERVAL)
    out = sh.search(Q, [0], NPROBE, KK)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), owners=owners, assigned=assigned, ids=out.ids,
             d=out.dists, cids=out.cids, n=out.counts, sc=out.scanned)
    sh.local.close()
    dist.destroy_process_group()


def test_sharded_inserts_two_processes_equal_sequential_reference(tmp_path):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    lists, Q, X, ids = _data()
    cids = list(range(NLIST))
    lists2, cents2, assigned = _sequential_inserts(lists, cids, X, ids, INTERVAL)
    flat = O.FlatIVF.from_lists(lists2, cents2, np.array(cids, np.int64))
    eids, edd, ecnt, _, esc = flat.search(Q, NPROBE, KK)
    id2cid = {int(i): c for (ii, _), c in zip(lists2, cids) for i in ii}
    res = [np.load(tmp_path / f"r{r}.npz") for r in range(2)]
    assert set(res[0]["owners"].tolist()) == {0, 1}
    for r in res:
        assert np.array_equal(r["assigned"], assigned)
        assert np.array_equal(r["ids"], eids)
        assert np.array_equal(r["d"].view(np.uint32), edd.view(np.uint32))
        assert np.array_equal(r["n"], ecnt)
        assert np.array_equal(r["sc"], esc)
        assert np.array_equal(r["cids"], np.vectorize(lambda i: id2cid.get(int(i), -1),
                                                      otypes=[np.int64])(eids))
