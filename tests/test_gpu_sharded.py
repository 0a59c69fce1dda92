"""Sharded search on the device, with R shards simulated
as R device indexes on one GPU: each owns the lists place_lists gives it and
holds the others as remote (centroid-only) lists; the R shard blocks are
merged by pk_merge_shards.  The merged answer must equal the single-index
device answer and the oracle bit for bit (ids, distance bits, hit cids,
scanned counts)."""

import numpy as np
import pytest

from oracle import oracle as O
from shard_oracle import merge_reference
from paper_2602_21477_b200.sharded import block_views, place_lists

pytestmark = pytest.mark.gpu


def _lists(seed, nlist, d, maxn):
    rng = np.random.default_rng(seed)
    cents = rng.normal(size=(nlist, d)).astype(np.float32)
    out, nid = [], 0
    for c in range(nlist):
        n = int(rng.integers(1, maxn))
        rows = (cents[c] + 0.5 * rng.normal(size=(n, d))).astype(np.float32)
        ids = rng.permutation(np.arange(nid, nid + n)).astype(np.int64)
        nid += n
        out.append((ids, rows))
    Q = (cents[rng.integers(0, nlist, 70)] + 0.5 * rng.normal(size=(70, d))).astype(np.float32)
    return out, Q


@pytest.mark.parametrize("R,d,nlist,nprobe,kk", [(2, 96, 40, 7, 10), (4, 384, 64, 16, 10),
                                                  (8, 128, 50, 50, 64), (3, 33, 30, 5, 1)])
def test_device_shards_merge_equals_single_index(R, d, nlist, nprobe, kk):
    from paper_2602_21477_b200 import DeviceIndex

    lists, Q = _lists(R * 100 + d, nlist, d, 700)
    cids = np.arange(1000, 1000 + nlist, dtype=np.int64)
    owners = place_lists([len(i) for i, _ in lists], R)
    single = DeviceIndex(d)
    cents = [single.create_list(int(c), 0, r, i) for c, (i, r) in zip(cids, lists)]
    shards = [DeviceIndex(d) for _ in range(R)]
    for j, (c, (i, r)) in enumerate(zip(cids, lists)):
        for s in range(R):
            if owners[j] == s:
                got = shards[s].create_list(int(c), 0, r, i)
                assert np.array_equal(got.view(np.uint32), cents[j].view(np.uint32))
            else:
                shards[s].add_remote_list(int(c), 0, cents[j])
    blocks = [sh.search_block(Q, [0], nprobe, kk) for sh in shards]
    B = len(Q)
    ids, dd, hc, cnt, sc = shards[0].merge_shards(np.concatenate(blocks), R, B, kk)
    ref = single.search(Q, [0], nprobe, kk)
    assert np.array_equal(ids, ref.ids)
    assert np.array_equal(dd.view(np.uint32), ref.dists.view(np.uint32))
    assert np.array_equal(hc, ref.cids)
    assert np.array_equal(cnt, ref.counts)
    assert np.array_equal(sc, ref.scanned)
    # the device merge equals the numpy restatement of _topk's merge
    parts = [block_views(b, B, kk) for b in blocks]
    r_ids, r_d, r_c, r_n, r_sc = merge_reference(parts, B, kk)
    assert np.array_equal(ids, r_ids) and np.array_equal(cnt, r_n) and np.array_equal(sc, r_sc)
    assert np.array_equal(hc, r_c)
    # and the oracle over the whole index
    flat = O.FlatIVF.from_lists(lists, np.stack(cents), cids)
    o_ids, o_d, o_n, _, o_sc = flat.search(Q, nprobe, kk)
    assert np.array_equal(ids, o_ids)
    assert np.array_equal(dd.view(np.uint32), o_d.view(np.uint32))
    assert np.array_equal(sc, o_sc)
    for ix in shards + [single]:
        ix.close()


def test_remote_list_rejects_append():
    from paper_2602_21477_b200 import DeviceIndex, UsageError

    ix = DeviceIndex(16)
    ix.add_remote_list(5, 0, np.ones(16, np.float32))
    with pytest.raises(UsageError):  # appends are queued: the error surfaces at the flush
        ix.append(5, np.ones((1, 16), np.float32), [1])
        ix.flush()
    assert ix.size(5) == 0
    ix.retire(5)
    ix.close()


def test_sharded_index_single_process_device_path():
    """ShardedIndex with world 1 (no process group): the product wrapper."""
    from paper_2602_21477_b200.sharded import ShardedIndex

    d, nlist = 64, 20
    lists, Q = _lists(9, nlist, d, 300)
    cids = list(range(nlist))
    sh = ShardedIndex(d)
    sh.load(cids, [0] * nlist, [len(i) for i, _ in lists], lambda i: lists[i][::-1])
    out = sh.search(Q, [0], 6, 10)
    cents = np.stack([O.centroid(r) for _, r in lists])
    flat = O.FlatIVF.from_lists(lists, cents, np.array(cids, np.int64))
    o_ids, o_d, o_n, _, o_sc = flat.search(Q, 6, 10)
    assert np.array_equal(out.ids, o_ids)
    assert np.array_equal(out.dists.view(np.uint32), o_d.view(np.uint32))
    assert np.array_equal(out.scanned, o_sc)


@pytest.mark.parametrize("R", [2, 3])
def test_device_dispatch_combine_equals_single_index(R):
    """Dispatch/combine (every rank brings its own batch): coarse on each
    rank's own queries, scan of the concatenated batch on every shard into
    per-origin blocks, 'all-to-all' (block r of every shard to rank r) and
    the device merge.  Shards built in global order share list handles."""
    from paper_2602_21477_b200 import DeviceIndex
    from paper_2602_21477_b200.sharded import block_offsets

    d, nlist, nprobe, kk = 128, 45, 9, 10
    lists, Q = _lists(77 + R, nlist, d, 600)
    Q = Q[:R * 20]
    B = 20
    cids = np.arange(500, 500 + nlist, dtype=np.int64)
    owners = place_lists([len(i) for i, _ in lists], R)
    single = DeviceIndex(d)
    cents = [single.create_list(int(c), 0, r, i) for c, (i, r) in zip(cids, lists)]
    shards = [DeviceIndex(d) for _ in range(R)]
    for j, (c, (i, r)) in enumerate(zip(cids, lists)):  # global order on every shard
        for s in range(R):
            if owners[j] == s:
                shards[s].create_list(int(c), 0, r, i)
            else:
                shards[s].add_remote_list(int(c), 0, cents[j])
    probes = [shards[r].search_coarse(Q[r * B:(r + 1) * B], [0], nprobe) for r in range(R)]
    for r in range(1, R):  # handles agree across shards
        assert np.array_equal(shards[0].search_coarse(Q[r * B:(r + 1) * B], [0], nprobe), probes[r])
    P = np.concatenate(probes)
    sent = [sh.search_probed(Q, P, kk, B) for sh in shards]
    bb = block_offsets(B, kk)["total"]
    ref = single.search(Q, [0], nprobe, kk)
    for r in range(R):
        recv = np.concatenate([sent[s][r * bb:(r + 1) * bb] for s in range(R)])
        ids, dd, hc, cnt, sc = shards[r].merge_shards(recv, R, B, kk)
        sl = slice(r * B, (r + 1) * B)
        assert np.array_equal(ids, ref.ids[sl])
        assert np.array_equal(dd.view(np.uint32), ref.dists[sl].view(np.uint32))
        assert np.array_equal(hc, ref.cids[sl])
        assert np.array_equal(cnt, ref.counts[sl])
        assert np.array_equal(sc, ref.scanned[sl])
    for ix in shards + [single]:
        ix.close()


def test_peer_combine_in_process_equals_single_index():
    """The fused combine (P2P stores into each origin's area + device flags),
    R ranks simulated in one process: two epochs, every rank's answers equal
    the single index's."""
    from paper_2602_21477_b200 import DeviceIndex
    import torch

    R, d, nlist, nprobe, kk, B = 3, 64, 36, 7, 10, 16
    lists, Q = _lists(5150, nlist, d, 500)
    cids = np.arange(nlist, dtype=np.int64) + 70
    owners = place_lists([len(i) for i, _ in lists], R)
    single = DeviceIndex(d)
    cents = [single.create_list(int(c), 0, r, i) for c, (i, r) in zip(cids, lists)]
    shards = [DeviceIndex(d) for _ in range(R)]
    for j, (c, (i, r)) in enumerate(zip(cids, lists)):
        for s in range(R):
            if owners[j] == s:
                shards[s].create_list(int(c), 0, r, i)
            else:
                shards[s].add_remote_list(int(c), 0, cents[j])
    for s, sh in enumerate(shards):
        sh.combine_create(R, s, B, kk)
    for s, sh in enumerate(shards):
        for g in range(R):
            if g != s:
                sh.combine_open(g, area_ptr=shards[g].combine_area())
    dev = torch.device("cuda", 0)
    for epoch in (1, 2):
        Qe = Q[(epoch - 1) * 8:(epoch - 1) * 8 + R * B] if epoch == 1 else Q[-R * B:]
        ref = single.search(Qe, [0], nprobe, kk)
        probes = [shards[r].search_coarse(Qe[r * B:(r + 1) * B], [0], nprobe) for r in range(R)]
        qa = torch.from_numpy(np.ascontiguousarray(Qe)).to(dev)
        pa = torch.from_numpy(np.concatenate(probes)).to(dev)
        for sh in shards:
            sh.combine_search_probed_device(qa, pa, epoch)
        for sh in shards:
            sh.sync()
        for r, sh in enumerate(shards):
            o_ids = torch.empty(B, kk, dtype=torch.int64, device=dev)
            o_d = torch.empty(B, kk, dtype=torch.float32, device=dev)
            o_c = torch.empty(B, kk, dtype=torch.int64, device=dev)
            o_n = torch.empty(B, dtype=torch.int32, device=dev)
            o_s = torch.empty(B, dtype=torch.int64, device=dev)
            sh.combine_merge_device(epoch, o_ids, o_d, o_c, o_n, o_s, timeout_s=5.0)
            sh.sync()
            assert sh.combine_status() == 0
            sl = slice(r * B, (r + 1) * B)
            assert np.array_equal(o_ids.cpu().numpy(), ref.ids[sl])
            assert np.array_equal(o_d.cpu().numpy().view(np.uint32), ref.dists[sl].view(np.uint32))
            assert np.array_equal(o_c.cpu().numpy(), ref.cids[sl])
            assert np.array_equal(o_n.cpu().numpy(), ref.counts[sl])
            assert np.array_equal(o_s.cpu().numpy(), ref.scanned[sl])
    # a merge for an epoch nobody produced times out instead of hanging
    o = [torch.empty(B, kk, dtype=torch.int64, device=dev), torch.empty(B, kk, dtype=torch.float32, device=dev),
         torch.empty(B, kk, dtype=torch.int64, device=dev), torch.empty(B, dtype=torch.int32, device=dev)]
    shards[0].combine_merge_device(99, *o, timeout_s=0.05)
    shards[0].sync()
    assert shards[0].combine_status() == 1
    for ix in shards + [single]:
        ix.close()
