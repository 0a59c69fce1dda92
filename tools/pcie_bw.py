"""Host<->device bandwidth of this box: one large pinned copy each way, and a
copy-engine copy split into N segments of S MB (the cold tier's per-list
staging shape)."""
import json
import time

import torch


def bw(fn, nbytes, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return round(nbytes * reps / (time.perf_counter() - t) / 1e9, 1)


n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
out = {"h2d_1GB": bw(lambda: d.copy_(h, non_blocking=True), n),
       "d2h_1GB": bw(lambda: h.copy_(d, non_blocking=True), n)}
for seg_mb in (1, 3, 16):
    seg = seg_mb << 20
    k = n // seg

    def segs():
        for i in range(k):
            d[i * seg:(i + 1) * seg].copy_(h[i * seg:(i + 1) * seg], non_blocking=True)

    out[f"h2d_{seg_mb}MB_segments"] = bw(segs, k * seg, 3)
print(json.dumps(out))
