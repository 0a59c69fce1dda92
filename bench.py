#!/usr/bin/env python3
"""Benchmark of the B200-native IVF search hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config auto|0|1|3] [--mode strong|weak]

A step is one batched search through the fused device path (coarse quantizer
on tcgen05 -> screened posting-list scan -> exact re-rank + top-k), exact
reference arithmetic.  Workloads (BASELINE.json configs, synthetic
unit-sphere fp32 rows, k 10):

  configs[0]  100K x 384, nlist 256,  nprobe 16, 32 queries per step
  configs[1]  1M x 768,   nlist 1024, nprobe 32, 256 queries per step
  configs[3]  10M x 768,  nlist 8192, nprobe 32, 256 queries per step

``--config auto`` (default): configs[1] on one GPU (the N=1 headline), and
configs[3] for N > 1.  configs[3] is STRONG scaling: the same 10M-vector
index at every N, its lists placed on the N ranks by size-balanced greedy
packing (centroids replicated), every rank answering the same 256-query
batch over its own lists, the per-shard top-k all-gathered (NCCL) and merged
on the device; N=1 is the whole index on one GPU.  ``--config 1 --mode weak``
keeps round 1's weak-scaling mode (every rank owns its own 1M shard and
brings its own batch; dispatch/combine with the combine fused into the scan's
write-out over NVLink P2P).

``--gpus N`` with N > 1 and no torchrun environment re-launches itself under
``torch.distributed.run`` with N local ranks.

Prints ONE JSON line (rank 0):

  value   device QPS with queries already resident in HBM (CUDA events on the
          index stream around exactly K steps, max over ranks)
  e2e     QPS through the public API with host buffers (pinned), H2D of the
          queries and D2H of the results inside the timed region
  roofline  the fused scan kernel: algorithmic bytes of the distinct posting
          lists each launch reads / its CUDA-event duration, against the
          measured HBM copy bandwidth (MEASURED_PEAKS.json); ``traffic`` is the
          ncu DRAM bytes of one scan launch of the SAME workload
          (profiles/scan_ncu_traffic.json), null when none was captured
  cpu_baseline  the C oracle port (oracle/, the parity checker) on one full
          step of queries, all host threads (rank 0)
  parity_vs_oracle  the same step's answers (ids, distance bits, probe sets)
          against the oracle over the single global index

The index is the same in both arms: rows and queries are drawn on the device
with seeded Philox generators (torch), each row goes to its nearest of nlist
seed rows (fp32 GEMM, TF32 off: a one-round k-means), rows are grouped by
list in row order; ``config.index_fingerprint`` hashes the list sizes and
ids so the two arms' lines can be compared.  ``--impl reference`` times the
oracle port alone (the reference is a pure-Python/numba package; its hot path
restated in C) on the same index and queries.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "search QPS at recall@10 (=CPU ref) + scan HBM GB/s, 1/2/4/8 B200"
UNIT = "queries/s"
E2E_DEPTH = int(os.environ.get("PK_BENCH_E2E_DEPTH", "4"))  # host batches in flight on the e2e path (<= 4 slots)

CONFIGS = {
    0: dict(n=100_000, d=384, nlist=256, nprobe=16, k=10, batch=32),
    1: dict(n=1_000_000, d=768, nlist=1024, nprobe=32, k=10, batch=256),
    3: dict(n=10_000_000, d=768, nlist=8192, nprobe=32, k=10, batch=256),
}
CHUNK = 1 << 17  # generator chunk (rows); chunk c is drawn from seed (seed, c)


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="auto", choices=["auto", "0", "1", "3"])
    p.add_argument("--mode", default="auto", choices=["auto", "strong", "weak"],
                   help="N>1: strong (one global index, default) or weak (one shard per rank)")
    p.add_argument("--rows", dest="n", type=int, default=None, help="index rows (global)")
    p.add_argument("--d", type=int, default=None)
    p.add_argument("--nlist", type=int, default=None)
    p.add_argument("--nprobe", type=int, default=None)
    p.add_argument("--k", type=int, default=None)
    p.add_argument("--batch", type=int, default=None)
    p.add_argument("--cpu-sample", type=int, default=0, help="oracle sample queries (0 = one step)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-parity", action="store_true")
    p.add_argument("--seed", type=int, default=0)
    return p.parse_args(argv)


def resolve(a, world: int):
    """Fill the workload from --config (explicit flags override)."""
    cfg = a.config
    if cfg == "auto":
        cfg = "1" if world == 1 else "3"
    a.cfg = int(cfg)
    base = CONFIGS[a.cfg]
    for key, v in base.items():
        if getattr(a, key) is None:
            setattr(a, key, v)
    a.named = all(getattr(a, key) == v for key, v in base.items())
    if a.mode == "auto":
        a.mode = "strong"
    if world == 1:
        a.mode = "strong"
    return a


def workload_name(a, world: int) -> str:
    tag = f"configs[{a.cfg}]" if a.named else f"custom (from configs[{a.cfg}])"
    n = f"{a.n / 1e6:g}M" if a.n >= 1_000_000 else f"{a.n // 1000}K"
    if a.mode == "weak" and world > 1:
        return (f"{tag} weak scaling: {world} x {n} x {a.d} fp32 shards (nlist {a.nlist} each, global "
                f"nlist {world * a.nlist}), nprobe {a.nprobe}, k {a.k}, {a.batch} queries per rank per step")
    s = (f"{tag}: {n} x {a.d} fp32 IVF, nlist {a.nlist}, nprobe {a.nprobe}, k {a.k}, "
         f"{a.batch} queries per step")
    if world > 1:
        s += f", lists placed on {world} GPUs (strong scaling: same index and batch at every N)"
    return s


# ---------------------------------------------------------------- self-launch
def maybe_relaunch(a):
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run."""
    if a.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


# ---------------------------------------------------------------- workload
def gen_rows(n, d, seed, dev, salt=0):
    """Unit-sphere fp32 rows (bench/workload.py:108-111 semantics: N(0, I)
    normalised) drawn on the device, chunk c from Philox seed (seed, salt, c)."""
    import torch

    out = torch.empty(n, d, dtype=torch.float32, device=dev)
    g = torch.Generator(device=dev)
    for c, i in enumerate(range(0, n, CHUNK)):
        m = min(CHUNK, n - i)
        g.manual_seed((seed * 1_000_003 + salt * 7_919 + c) & 0x7FFFFFFFFFFF)
        x = torch.randn(m, d, generator=g, device=dev, dtype=torch.float32)
        out[i:i + m] = x / torch.linalg.vector_norm(x, dim=1, keepdim=True)
    return out


def gen_queries(X, count, seed, dev):
    """Half perturbed base rows (x + 0.01 N(0, I)), half fresh unit vectors,
    interleaved by a seeded permutation (bench/workload.py:114-125)."""
    import torch

    n, d = X.shape
    g = torch.Generator(device=dev)
    g.manual_seed(seed * 31 + 17)
    h = count // 2
    pick = torch.randint(0, n, (h,), generator=g, device=dev)
    near = X[pick] + 0.01 * torch.randn(h, d, generator=g, device=dev)
    fresh = gen_rows(count - h, d, seed, dev, salt=99)
    Q = torch.cat([near, fresh])
    perm = torch.randperm(count, generator=g, device=dev)
    return Q[perm].contiguous()


def build_partition(a, dev):
    """The IVF partition both arms use: seeded rows, nlist seed rows, every row
    to its nearest seed (fp32 GEMM, TF32 off, ties to the lower seed index).
    Returns (X [n, d] on dev, order [n] i64 = rows grouped by list in row
    order, lens [nlist] i64, offs [nlist] i64)."""
    import torch

    torch.backends.cuda.matmul.allow_tf32 = False
    X = gen_rows(a.n, a.d, a.seed, dev)
    g = torch.Generator(device=dev)
    g.manual_seed(a.seed * 13 + 104729)
    seeds = torch.randperm(a.n, generator=g, device=dev)[:a.nlist].sort().values
    C = X[seeds].contiguous()
    cn = (C * C).sum(1)
    labels = torch.empty(a.n, dtype=torch.int64, device=dev)
    step = 1 << 18
    for i in range(0, a.n, step):
        blk = X[i:i + step]
        labels[i:i + len(blk)] = torch.argmin(cn[None, :] - 2.0 * (blk @ C.T), dim=1)
    del C
    order = torch.argsort(labels, stable=True)
    lens = torch.bincount(labels, minlength=a.nlist).cpu().numpy().astype(np.int64)
    del labels
    offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    torch.cuda.synchronize(dev)
    return X, order, lens, offs


def fingerprint(lens, order_h):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(lens, np.int64).tobytes())
    h.update(np.ascontiguousarray(order_h[:: max(1, len(order_h) // 65536)], np.int64).tobytes())
    return h.hexdigest()[:16]


def host_index(X, order, lens, offs):
    """Rows grouped by list, copied to host in chunks, plus the oracle's own
    centroids (Cluster.recompute_stats arithmetic, ref/clusters.py:111-118)."""
    from oracle import oracle as O

    n, d = X.shape
    rows_h = np.empty((n, d), dtype=np.float32)
    step = 1 << 20
    for i in range(0, n, step):
        rows_h[i:i + step] = X[order[i:i + step]].cpu().numpy()
    ids_h = order.cpu().numpy().astype(np.int64)
    live = np.nonzero(lens > 0)[0]
    cents = np.stack([O.centroid(rows_h[offs[c]:offs[c] + lens[c]]) for c in live])
    flat = O.FlatIVF(rows_h, ids_h, offs[live], lens[live], cents, live.astype(np.int64))
    return flat, ids_h, live


# ---------------------------------------------------------------- helpers
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_read_peak():
    """Read-only streaming peak measured on this hardware
    (tools/microbench/hbm_read.cu -> profiles/hbm_read_peak.json)."""
    p = os.path.join(ROOT, "profiles", "hbm_read_peak.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["read_gbs"])
    return None


def load_traffic(key):
    """ncu DRAM bytes of one scan launch of this workload, or None."""
    p = os.path.join(ROOT, "profiles", "scan_ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(key)
    return None


class ClockSampler:
    """NVML sampling of SM clocks and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device=0, period=0.005):
        self.samples, self.reasons = [], set()
        self.period = period
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def config_block(a, world, fp, extra=None):
    c = {"workload": workload_name(a, world), "n": a.n, "d": a.d, "nlist": a.nlist,
         "nprobe": a.nprobe, "k": a.k, "batch": a.batch, "index_fingerprint": fp,
         "index": ("seeded Philox unit-sphere rows on the device, nlist seed rows, nearest-seed "
                   "assignment (fp32 GEMM), lists in row order; same in both arms"),
         "l2": (f"inputs larger than L2 (index {a.n * (4 * a.d + 8) / 1e9:.2f} GB vs 126 MB L2; "
                "each batch reads most of its lists)")}
    if extra:
        c.update(extra)
    return c


def gather_max(dist, dev, v):
    import torch

    if dist is None:
        return v
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- reference arm
def run_reference(a):
    """The reference's CPU path (the C restatement of ref/kernels.py +
    ref/graph.py at exhaustive ef + ref/engine.py:319-426, oracle/) over the
    same index and queries; rank 0 alone, all host threads, each step a
    bounded sample of that step's queries."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    resolve(a, world)
    if int(os.environ.get("RANK", "0")) != 0:
        return
    import torch

    from oracle import oracle as O  # noqa: F401  (the checker is the timed CPU path here)

    dev = torch.device("cuda", 0)
    t_build = time.perf_counter()
    X, order, lens, offs = build_partition(a, dev)
    Qall = gen_queries(X, (a.warmup + a.steps) * a.batch, a.seed, dev).cpu().numpy()
    flat, ids_h, live = host_index(X, order, lens, offs)
    fp = fingerprint(lens, ids_h)
    del X, order
    torch.cuda.empty_cache()
    build_s = time.perf_counter() - t_build
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    flat.search(Qall[:threads], a.nprobe, a.k, threads=threads)
    per_q = (time.perf_counter() - t0) / threads
    # bounded sample: the whole run stays near a minute of CPU time
    sample = max(1, min(a.batch, int(60.0 / max(1, a.steps) / max(per_q, 1e-6))))
    if a.cpu_sample:
        sample = a.cpu_sample
    for w in range(a.warmup):
        flat.search(Qall[w * a.batch: w * a.batch + sample], a.nprobe, a.k, threads=threads)
    t_total = 0.0
    for s in range(a.steps):
        lo = (a.warmup + s) * a.batch
        t0 = time.perf_counter()
        flat.search(Qall[lo: lo + sample], a.nprobe, a.k, threads=threads)
        t_total += time.perf_counter() - t0
    qps = a.steps * sample / t_total
    line = {
        "impl": "reference", "metric": METRIC, "value": qps, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1000.0 * t_total / a.steps,
        "higher_is_better": True, "scaling": "strong" if a.mode == "strong" else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_block(a, 1, fp, {"sample_queries_per_step": sample}),
        "cpu_baseline": {"value": qps, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{sample} of each step's {a.batch} queries, C oracle "
                                   f"(oracle/pancake_oracle.c) on {threads} threads"},
        "e2e": {"value": qps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "build_s": build_s,
        "note": ("CPU path of the reference restated in C (the reference itself is a numba "
                 "package, SURVEY.md section 8c); index built on the device (setup, untimed) "
                 "exactly as in the GPU arm"),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def run_ours(a):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    resolve(a, world)
    # PK_BENCH_SHARE_GPU=1: every rank on cuda:0 over gloo -- only to exercise
    # the multi-rank code path on a one-GPU box; never a bench number
    share = os.environ.get("PK_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    from paper_2602_21477_b200 import DeviceIndex
    from paper_2602_21477_b200 import _native as N
    from paper_2602_21477_b200 import build as B
    from paper_2602_21477_b200.sharded import ShardedIndex, block_offsets

    if rank == 0:
        B.build()
    if dist:
        dist.barrier()
    N.load()

    weak = world > 1 and a.mode == "weak"
    t_build = time.perf_counter()
    if weak:  # rank r owns its own a.n-row shard (seed + r)
        a_r = argparse.Namespace(**vars(a))
        a_r.seed = a.seed + rank
        X, order, lens, offs = build_partition(a_r, dev)
    else:  # every rank derives the same global partition
        X, order, lens, offs = build_partition(a, dev)
    Qall = gen_queries(X, (a.warmup + a.steps) * a.batch, a.seed + (1000 * rank if weak else 0), dev)
    Qall_h = Qall.cpu().numpy()
    Qall = Qall.view(a.warmup + a.steps, a.batch, a.d)
    live = np.nonzero(lens > 0)[0]
    kk = a.k
    # rank 0's host copy of the global index: the oracle's input (cpu_baseline, parity)
    flat = None
    if rank == 0 and not a.no_parity:
        flat, ids_h, _ = host_index(X, order, lens, offs)
        fp = fingerprint(lens, ids_h)
        del ids_h
    else:
        fp = fingerprint(lens, order.cpu().numpy())

    def fetch_rows(c):
        sel = order[offs[c]:offs[c] + lens[c]]
        return X[sel].contiguous(), sel.contiguous()

    sh = None
    if world == 1:
        ix = DeviceIndex(a.d, 0, local, reserve_rows=int(a.n * 1.26) + 32 * a.nlist + 4096,
                         reserve_lists=a.nlist)
        for c in live:
            rows, ids = fetch_rows(c)
            ix.create_list(int(c), 0, rows, ids)
        gl_lens = lens[live]
        mine = np.ones(len(live), dtype=bool)
    elif weak:
        # global list table: rank r's list c is cid r * nlist + c, owned by r
        lens_all = torch.empty(world * a.nlist, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(lens_all, torch.from_numpy(lens).to(dev))
        lens_all = lens_all.cpu().numpy().reshape(world, a.nlist)
        gl = [(r, c) for r in range(world) for c in range(a.nlist) if lens_all[r, c] > 0]
        sh = ShardedIndex(a.d, 0, local, reserve_rows=int(a.n * 1.26) + 32 * a.nlist + 4096,
                          reserve_lists=a.nlist * world)
        ix = sh.local
        sh.load([r * a.nlist + c for r, c in gl], [0] * len(gl),
                [int(lens_all[r, c]) for r, c in gl], lambda i: fetch_rows(gl[i][1]),
                owners=[r for r, _ in gl])
        gl_lens = np.array([int(lens_all[r, c]) for r, c in gl], dtype=np.int64)
        mine = np.array([r == rank for r, _ in gl])
    else:
        share_rows = int(a.n / world * 1.3) + 32 * a.nlist + 4096
        sh = ShardedIndex(a.d, 0, local, reserve_rows=share_rows, reserve_lists=a.nlist)
        ix = sh.local
        owners = sh.load(live.tolist(), [0] * len(live), lens[live].tolist(),
                         lambda i: fetch_rows(live[i]))
        gl_lens = lens[live]
        mine = owners == rank
    del X, order
    torch.cuda.synchronize()
    torch.cuda.empty_cache()  # the index arena is cudaMalloc'd outside torch's cache
    build_s = time.perf_counter() - t_build

    codes = torch.zeros(1, dtype=torch.int32, device=dev)
    o_ids = torch.empty(a.batch, kk, dtype=torch.int64, device=dev)
    o_d = torch.empty(a.batch, kk, dtype=torch.float32, device=dev)
    o_c = torch.empty(a.batch, kk, dtype=torch.int64, device=dev)
    o_n = torch.empty(a.batch, dtype=torch.int32, device=dev)
    o_s = torch.empty(a.batch, dtype=torch.int64, device=dev)
    stream = torch.cuda.ExternalStream(ix.stream_handle(), device=dev)
    bb = block_offsets(a.batch, kk)["total"]
    bufs = None
    combine = None
    if weak:
        bufs = {"probe": torch.empty(a.batch, a.nprobe, dtype=torch.int32, device=dev),
                "q_all": torch.empty(world * a.batch, a.d, dtype=torch.float32, device=dev),
                "probe_all": torch.empty(world * a.batch, a.nprobe, dtype=torch.int32, device=dev),
                "send": torch.empty(world * bb, dtype=torch.uint8, device=dev),
                "recv": torch.empty(world * bb, dtype=torch.uint8, device=dev)}
        # combine: results written straight into their origin rank's HBM over
        # NVLink (CUDA IPC + device flags, PK_COMBINE=peer, default) or an NCCL
        # all-to-all (PK_COMBINE=nccl, or when the peer mapping cannot be set up)
        combine = os.environ.get("PK_COMBINE", "peer")
        if combine == "peer":
            ok = 1
            try:
                sh.setup_peer_combine(a.batch, kk)
            except Exception as exc:  # no P2P mapping between these devices
                print(f"rank {rank}: peer combine unavailable ({exc})", file=sys.stderr)
                ok = 0
            flag = torch.tensor([ok], dtype=torch.int32, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 0:
                combine = "nccl"
    elif sh is not None:
        bufs = {"block": torch.empty(bb, dtype=torch.uint8, device=dev),
                "gathered": torch.empty(world * bb, dtype=torch.uint8, device=dev)}

    def step(s):
        if sh is None:
            ix.search_device(Qall[s], codes, a.nprobe, kk, o_ids, o_d, o_c, o_n, o_s)
            return
        with torch.cuda.stream(stream):
            if weak and combine == "peer":
                sh.search_dispatch_peer(Qall[s], codes, a.nprobe, kk, bufs, o_ids, o_d, o_c, o_n, o_s)
            elif weak:
                sh.search_dispatch_device(Qall[s], codes, a.nprobe, kk, bufs, o_ids, o_d, o_c, o_n, o_s)
            else:
                sh.search_device(Qall[s], codes, a.nprobe, kk, bufs["block"], bufs["gathered"],
                                 o_ids, o_d, o_c, o_n, o_s)

    for w in range(a.warmup):
        step(w)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            ev0.record(stream)
        for s in range(a.steps):
            step(a.warmup + s)
        with torch.cuda.stream(stream):
            ev1.record(stream)
        torch.cuda.synchronize()
    ms = gather_max(dist, dev, ev0.elapsed_time(ev1))
    # stage breakdown + the scan kernel's own duration (roofline): a separate
    # pass over the same batches with per-stage events (kept out of the timed
    # loop above, whose value carries no profiling overhead)
    if dist:
        dist.barrier()
    ix.profile_begin()
    for s in range(a.steps):
        step(a.warmup + s)
    torch.cuda.synchronize()
    stage_ms, ncalls = ix.profile_end()
    if weak and combine == "peer" and ix.combine_status() != 0:
        raise RuntimeError("peer combine timed out waiting for a rank's results")
    queries_per_step = world * a.batch if weak else a.batch
    qps = a.steps * queries_per_step / (ms / 1000.0)

    # ---- roofline of the fused scan: algorithmic bytes of the distinct local
    # lists each scan launch reads (the probe sets of the same batches)
    row_bytes = 4 * a.d + 8
    alg_bytes = []
    for s in range(a.steps):
        if weak:
            step(a.warmup + s)
            torch.cuda.synchronize()
            pa = bufs["probe_all"].cpu().numpy()
            pr = np.unique(pa[pa >= 0])  # list handles = global registration order
        else:
            pr = np.unique(ix.search_coarse(Qall_h[(a.warmup + s) * a.batch:(a.warmup + s + 1) * a.batch],
                                            [0], a.nprobe))
            pr = pr[pr >= 0]
        alg_bytes.append(float(gl_lens[pr][mine[pr]].sum()) * row_bytes)
    pool = None
    try:
        if sh is None:
            ix.search(Qall_h[a.warmup * a.batch:(a.warmup + 1) * a.batch], [0], a.nprobe, kk)
        B_last = a.batch * (world if weak else 1)
        pc = ix.pool_counts(B_last)
        pool = {"mean": float(pc.mean()), "max": int(pc.max()), "p50": float(np.median(pc)),
                "rows_reranked_per_step": int(pc.sum())}
        if sh is None:
            cc = ix.coarse_counts(a.batch)
            pool["coarse_lists_reranked"] = {"mean": float(cc.mean()), "max": int(cc.max())}
        rc = ix.rerank_counts(B_last)
        pool["rows_reranked_exactly"] = {"mean": float(rc.mean()), "max": int(rc.max())}
    except Exception:
        pass
    scan_ms = stage_ms["scan"] / max(ncalls, 1)
    achieved = float(np.mean(alg_bytes)) / (scan_ms / 1000.0) / 1e9
    peak, peak_src = load_peaks()
    read_peak = load_read_peak()
    traffic_key = f"configs[{a.cfg}]" + (f" x{world} {a.mode}" if world > 1 else "")
    traffic = load_traffic(traffic_key) if a.named else None

    # ---- e2e through the public API with host buffers (pinned queries in,
    # results out, every step)
    e2e = None
    if not a.no_e2e:
        Qpin = torch.from_numpy(Qall_h).pin_memory().numpy().reshape(a.warmup + a.steps, a.batch, a.d)

        def host_run(first, count):
            """count host batches: N=1 keeps E2E_DEPTH in flight (submit
            batch s+3, then collect batch s: the H2D and host work of the next
            batches overlap the device pass, and the next batch's front half
            is queued before the current scan ends); N>1 runs the sharded
            host path."""
            if weak:
                for s in range(first, first + count):
                    sh.search_dispatch(Qpin[s], [0], a.nprobe, kk)
                return
            if sh is not None:
                for s in range(first, first + count):
                    sh.search(Qpin[s], [0], a.nprobe, kk)
                return
            inflight = []
            ht = os.environ.get("PK_BENCH_HOST_TIMES")  # host seconds inside submit / collect
            tsub = tcol = 0.0
            for s in range(first, first + count):
                t0_ = time.perf_counter()
                inflight.append(ix.search_submit(Qpin[s], [0], a.nprobe, kk))
                t1_ = time.perf_counter()
                tsub += t1_ - t0_
                if len(inflight) == E2E_DEPTH:
                    ix.search_collect(inflight.pop(0))
                    tcol += time.perf_counter() - t1_
            for t in inflight:
                ix.search_collect(t)
            if ht and count > 10:
                print(f"e2e host us/batch: submit {1e6 * tsub / count:.1f} collect {1e6 * tcol / count:.1f}",
                      file=sys.stderr)

        # every async slot touched (its buffers allocated) before the timed region
        host_run(0, min(a.warmup + a.steps, max(a.warmup, 2 * E2E_DEPTH)))
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        host_run(a.warmup, a.steps)
        e2e_s = gather_max(dist, dev, time.perf_counter() - t0)
        path = (f"DeviceIndex.search_submit / search_collect (pk_search_submit / pk_search_collect "
                f"C-ABI, {E2E_DEPTH} batches in flight: batch s+{E2E_DEPTH - 1} submitted before batch s is "
                "collected)"
                if sh is None else
                "ShardedIndex.search_dispatch (pk_search_coarse / NCCL / pk_search_probed / "
                "pk_merge_shards)" if weak else
                "ShardedIndex.search (pk_search into a shard block / all-gather / pk_merge_shards)")
        e2e = {"value": a.steps * queries_per_step / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": a.batch * a.d * 4,
               "d2h_bytes_per_step": a.batch * (kk * (8 + 4 + 8) + 4 + 8),
               "path": path + ", pinned host query buffer, every step's results read back to host"}

    # ---- CPU baseline (oracle port) + parity on one full timed step, rank 0:
    # the oracle runs over the single global index
    cpu = parity = None
    if rank == 0 and flat is not None:
        threads = os.cpu_count() or 1
        sample = a.cpu_sample or a.batch
        s0 = a.warmup
        Qs = Qall_h[s0 * a.batch: s0 * a.batch + sample]
        t0 = time.perf_counter()
        r_ids, r_d, r_n, r_p, r_sc = flat.search(Qs, a.nprobe, kk, threads=threads)
        t_cpu = time.perf_counter() - t0
        cpu = {"value": sample / t_cpu, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{sample} queries of timed step 0 (the whole step), C oracle "
                         f"(oracle/pancake_oracle.c), {threads} threads"}
        parity = {"queries": sample}
        if weak:  # rank 0's oracle holds its own shard only; answers span all shards
            step(s0)
            torch.cuda.synchronize()
            parity = {"note": "weak mode: no single-index oracle on rank 0 (see strong mode)"}
        elif sh is None:
            g = ix.search(Qs, [0], a.nprobe, kk, want_probe=True)
            parity["probe_mismatch"] = int((g.probe != r_p).sum())
            g_ids, g_d, g_sc = g.ids, g.dists, g.scanned
        else:
            step(s0)
            torch.cuda.synchronize()
            g_ids, g_d, g_sc = (o_ids.cpu().numpy()[:sample], o_d.cpu().numpy()[:sample],
                                o_s.cpu().numpy()[:sample])
        if not weak:
            parity["id_mismatch"] = int((g_ids != r_ids).sum())
            parity["dist_bit_mismatch"] = int((g_d.view(np.uint32) != r_d.view(np.uint32)).sum())
            parity["scanned_mismatch"] = int((g_sc != r_sc).sum())
    elif sh is not None:
        step(a.warmup)  # keep the collectives matched with rank 0's parity step
        torch.cuda.synchronize()

    if rank == 0:
        if sh is None:
            per_step = 6  # qprep, coarse_tc, coarse_pick (+ routing), route_items, scan_tc, rerank_merge
        elif weak:
            per_step = 10
        else:
            per_step = 7  # the 6 search kernels writing a shard block + shard_merge
        line = {
            "metric": METRIC, "value": qps, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
            "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": config_block(a, world, fp, {
                "parallelism": f"list-sharded x{world}" + (
                    "" if world == 1 else
                    ", dispatch (NCCL all-gather of queries + list handles) / combine ("
                    + ("per-shard top-k written into the origin rank's HBM over NVLink P2P, "
                       "device flags, device merge" if combine == "peer" else
                       "NCCL all-to-all of per-shard top-k, device merge") + ")" if weak else
                    ", replicated centroids and batch, NCCL all-gather of per-shard top-k, "
                    "device merge"),
                "comm": ("gloo, all ranks on cuda:0 (PK_BENCH_SHARE_GPU=1: code-path check, "
                         "not a bench number)" if share else "nccl") if world > 1 else None}),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                         "traffic_source": traffic.get("source") if traffic else
                         "no ncu capture of this workload",
                         "kernel": "scan_tc_kernel<SQ_L2> (TMA-fed tcgen05 TF32-screened posting-list "
                                   "scan + per-list top-k bounds)",
                         "algorithmic_bytes_per_launch": float(np.mean(alg_bytes)),
                         "kernel_ms_per_launch": scan_ms, "peak_source": peak_src,
                         "read_only_peak": read_peak,
                         "frac_of_read_only_peak": (achieved / read_peak) if read_peak else None},
            "stage_ms_per_step": {k_: v / max(ncalls, 1) for k_, v in stage_ms.items()},
            "gpu_launches": a.steps * per_step,
            "clocks": clk.summary(),
            "e2e": e2e, "cpu_baseline": cpu, "parity_vs_oracle": parity, "build_s": build_s,
            "screen_candidates_per_query": pool,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    ix.close()


def main():
    a = parse()
    maybe_relaunch(a)
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
