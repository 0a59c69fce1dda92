"""The fused peer combine across two PROCESSES (CUDA IPC handles exchanged over
a gloo process group, both ranks on cuda:0 of this one-GPU box): each rank
scans its own lists for the gathered batch and writes every origin's results
into that origin's HBM area through the IPC mapping; the merge acquires the
flags.  Producers are synchronised before the merges so the check does not
depend on two contexts time-slicing one GPU."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch
    import torch.distributed as dist

    from paper_2602_21477_b200 import DeviceIndex
    from paper_2602_21477_b200.sharded import place_lists
    from test_gpu_sharded import _lists

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    d, nlist, nprobe, kk, B = 48, 30, 6, 8, 12
    lists, Q = _lists(777, nlist, d, 400)
    cids = np.arange(nlist, dtype=np.int64)
    owners = place_lists([len(i) for i, _ in lists], world)
    single = DeviceIndex(d)
    cents = [single.create_list(int(c), 0, r, i) for c, (i, r) in zip(cids, lists)]
    ix = DeviceIndex(d)
    for j, (c, (i, r)) in enumerate(zip(cids, lists)):
        if owners[j] == rank:
            ix.create_list(int(c), 0, r, i)
        else:
            ix.add_remote_list(int(c), 0, cents[j])
    h = ix.combine_create(world, rank, B, kk)
    handles = [None] * world
    dist.all_gather_object(handles, h)
    for r in range(world):
        if r != rank:
            ix.combine_open(r, handle=handles[r])
    ok = True
    for epoch in (1, 2, 3):
        Qe = Q[epoch * 3:epoch * 3 + world * B]
        mine = Qe[rank * B:(rank + 1) * B]
        probe = ix.search_coarse(mine, [0], nprobe)
        allp = [None] * world
        dist.all_gather_object(allp, probe)
        qa = torch.from_numpy(np.ascontiguousarray(Qe)).to(dev)
        pa = torch.from_numpy(np.concatenate(allp)).to(dev)
        ix.combine_search_probed_device(qa, pa, epoch)
        ix.sync()
        dist.barrier()
        o_ids = torch.empty(B, kk, dtype=torch.int64, device=dev)
        o_d = torch.empty(B, kk, dtype=torch.float32, device=dev)
        o_c = torch.empty(B, kk, dtype=torch.int64, device=dev)
        o_n = torch.empty(B, dtype=torch.int32, device=dev)
        o_s = torch.empty(B, dtype=torch.int64, device=dev)
        ix.combine_merge_device(epoch, o_ids, o_d, o_c, o_n, o_s, timeout_s=10.0)
        ix.sync()
        ref = single.search(mine, [0], nprobe, kk)
        ok &= ix.combine_status() == 0
        ok &= np.array_equal(o_ids.cpu().numpy(), ref.ids)
        ok &= np.array_equal(o_d.cpu().numpy().view(np.uint32), ref.dists.view(np.uint32))
        ok &= np.array_equal(o_c.cpu().numpy(), ref.cids)
        ok &= np.array_equal(o_s.cpu().numpy(), ref.scanned)
        dist.barrier()
    with open(os.path.join(outdir, f"ok{rank}"), "w") as f:
        f.write("1" if ok else "0")
    dist.barrier()
    ix.close()
    single.close()
    dist.destroy_process_group()


def test_peer_combine_two_processes(tmp_path):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "ok0").read_text() == "1"
    assert (tmp_path / "ok1").read_text() == "1"
