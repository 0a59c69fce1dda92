"""Host enqueue cost vs device time of the device-pointer search at small
batches (is the step launch/host bound?).  Random clustered index of n x d."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2602_21477_b200 import DeviceIndex  # noqa: E402


def main(n=100_000, d=384, nlist=256, nprobe=16, kk=10):
    rng = np.random.default_rng(0)
    cent = rng.normal(size=(nlist, d)).astype(np.float32)
    lab = rng.integers(0, nlist, n)
    X = (cent[lab] + 0.5 * rng.normal(size=(n, d))).astype(np.float32)
    ix = DeviceIndex(d, 0, 0, reserve_rows=n + 1024, reserve_lists=nlist)
    for c in range(nlist):
        m = np.nonzero(lab == c)[0]
        ix.create_list(c, 0, X[m], m.astype(np.int64))
    dev = torch.device("cuda", 0)
    codes = torch.zeros(1, dtype=torch.int32, device=dev)
    out = {}
    for B in (1, 32, 256):
        Q = torch.from_numpy(rng.normal(size=(B, d)).astype(np.float32)).to(dev)
        o = (torch.empty(B, kk, dtype=torch.int64, device=dev), torch.empty(B, kk, device=dev),
             torch.empty(B, kk, dtype=torch.int64, device=dev), torch.empty(B, dtype=torch.int32, device=dev),
             torch.empty(B, dtype=torch.int64, device=dev))
        for _ in range(20):
            ix.search_device(Q, codes, nprobe, kk, *o)
        torch.cuda.synchronize()
        N = 500
        t0 = time.perf_counter()
        for _ in range(N):
            ix.search_device(Q, codes, nprobe, kk, *o)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        # the bare C-ABI call with pointers precomputed (no Python wrapper)
        from paper_2602_21477_b200 import _native as NN
        f = NN.lib().pk_search
        h = ix._h
        args = (Q.data_ptr(), B, codes.data_ptr(), 1, nprobe, kk, o[0].data_ptr(), o[1].data_ptr(),
                o[2].data_ptr(), o[3].data_ptr(), None, o[4].data_ptr(), NN.PK_DEVICE_PTRS)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        for _ in range(N):
            f(h, *args)
        t4 = time.perf_counter()
        torch.cuda.synchronize()
        out[f"B={B}"] = {"host_us_per_call": round((t1 - t0) / N * 1e6, 1),
                         "wall_us_per_call": round((t2 - t0) / N * 1e6, 1),
                         "abi_host_us_per_call": round((t4 - t3) / N * 1e6, 1)}
    print(json.dumps(out))
    ix.close()


if __name__ == "__main__":
    main()
