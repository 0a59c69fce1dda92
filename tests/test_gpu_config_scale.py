"""Parity at the BASELINE shapes: every query of whole
search batches at configs[1] (1M x 768, nlist 1024, nprobe 32, k 10, batch
256) and a sample at configs[3] (10M x 768, nlist 8192) on one GPU, against
the oracle over the same index -- ids, fp32 distance bits, probe sets and
scanned counts.  The index is bench.py's (seeded device rows, nearest-seed
partition), so these are the bench's own workloads; the device path is the
one the bench times (device-pointer searches, front-half overlap between
consecutive batches) and the host C-ABI path."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(cfg, nq_steps):
    import argparse

    import torch

    import bench
    from paper_2602_21477_b200 import DeviceIndex

    a = bench.resolve(argparse.Namespace(config=str(cfg), mode="auto", n=None, d=None, nlist=None,
                                         nprobe=None, k=None, batch=None, seed=0), 1)
    dev = torch.device("cuda", 0)
    X, order, lens, offs = bench.build_partition(a, dev)
    Q = bench.gen_queries(X, nq_steps * a.batch, 3, dev)
    flat, _, live = bench.host_index(X, order, lens, offs)
    ix = DeviceIndex(a.d, 0, 0, reserve_rows=int(a.n * 1.26) + 32 * a.nlist + 4096,
                     reserve_lists=a.nlist)
    for c in live:
        sel = order[offs[c]:offs[c] + lens[c]]
        ix.create_list(int(c), 0, X[sel].contiguous(), sel.contiguous())
    del X, order
    torch.cuda.empty_cache()
    return a, ix, flat, Q


def _device_batches(ix, a, Q):
    """Consecutive device-pointer searches (the bench's step: the next
    batch's front half overlaps this batch's scan)."""
    import torch

    dev = Q.device
    codes = torch.zeros(1, dtype=torch.int32, device=dev)
    nb = Q.shape[0] // a.batch
    outs = []
    for s in range(nb):
        o = (torch.empty(a.batch, a.k, dtype=torch.int64, device=dev),
             torch.empty(a.batch, a.k, dtype=torch.float32, device=dev),
             torch.empty(a.batch, a.k, dtype=torch.int64, device=dev),
             torch.empty(a.batch, dtype=torch.int32, device=dev),
             torch.empty(a.batch, dtype=torch.int64, device=dev))
        ix.search_device(Q[s * a.batch:(s + 1) * a.batch], codes, a.nprobe, a.k, *o)
        outs.append(o)
    torch.cuda.synchronize()
    return [tuple(t.cpu().numpy() for t in o) for o in outs]


def _check(got, want, tag):
    ids, d, _, n, sc = got
    r_ids, r_d, r_n, _, r_sc = want
    assert np.array_equal(ids, r_ids), tag
    assert np.array_equal(d.view(np.uint32), r_d.view(np.uint32)), tag
    assert np.array_equal(n, r_n), tag
    assert np.array_equal(sc, r_sc), tag


def test_configs1_whole_batches():
    a, ix, flat, Q = _setup(1, 3)
    Qh = Q.cpu().numpy()
    got = _device_batches(ix, a, Q)
    for s, g in enumerate(got):
        Qs = Qh[s * a.batch:(s + 1) * a.batch]
        want = flat.search(Qs, a.nprobe, a.k, threads=16)
        _check(g, want, f"device batch {s}")
        h = ix.search(Qs, [0], a.nprobe, a.k, want_probe=True)  # host C-ABI path
        assert np.array_equal(h.probe, want[3])
        _check((h.ids, h.dists, h.cids, h.counts, h.scanned), want, f"host batch {s}")
    ix.close()


def test_configs3_sample_one_gpu():
    a, ix, flat, Q = _setup(3, 1)
    Qh = Q.cpu().numpy()
    got = _device_batches(ix, a, Q)[0]
    sample = np.r_[0:48, a.batch - 16:a.batch]  # perturbed-row and fresh queries alike
    want = flat.search(Qh[sample], a.nprobe, a.k, threads=16)
    _check(tuple(x[sample] for x in got), want, "configs[3] sample")
    ix.close()
