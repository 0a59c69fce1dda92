#!/usr/bin/env python3
"""Benchmark of the B200-native IVF search hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one batched search: 256 queries against the configs[1] index
(1M x 768 fp32 unit-sphere vectors, nlist 1024, nprobe 32, k 10), exact
reference arithmetic.  Prints ONE JSON line (rank 0).

  value   device QPS with queries already resident in HBM (CUDA events on the
          index stream around exactly K steps, max over ranks)
  e2e     QPS through the C-ABI with host buffers (pinned), H2D of the queries
          and D2H of the results inside the timed region
  roofline  the fused scan kernel: algorithmic bytes of the distinct posting
          lists each batch reads / its CUDA-event duration, against the
          measured HBM copy bandwidth (MEASURED_PEAKS.json)
  cpu_baseline  the C oracle port (oracle/, the parity checker) on a bounded
          sample of the same queries, all host threads

--impl reference times that oracle port alone (the reference itself is a Python
package; its hot path restated in C is the CPU implementation of the path).
Multi-GPU (torchrun, N>1): weak scaling -- every rank owns a 1M x 768 shard of
an N-million-vector index (nlist 1024 N, lists sharded by rank, centroids
replicated) and brings its own 256 queries per step.  Dispatch: each rank runs
the coarse stage on its batch, the queries and their list handles are
all-gathered (NCCL); every rank scans its own lists for all N*256 queries;
combine: the per-shard top-k blocks go back to their origin rank (NCCL
all-to-all) and are merged on the device.
"""

from __future__ import annotations

import argparse
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


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--rows", dest="n", type=int, default=1_000_000, help="rows per GPU")
    p.add_argument("--d", type=int, default=768)
    p.add_argument("--nlist", type=int, default=1024)
    p.add_argument("--nprobe", type=int, default=32)
    p.add_argument("--k", type=int, default=10)
    p.add_argument("--batch", type=int, default=256)
    p.add_argument("--kmeans-iters", type=int, default=2)
    p.add_argument("--cpu-sample", type=int, default=0, help="oracle sample queries (0 = auto)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--seed", type=int, default=0)
    return p.parse_args()


def workload_name(a, world: int = 1) -> str:
    """The BASELINE config these arguments describe (configs[1] by default)."""
    shape = (a.n, a.d, a.nlist, a.nprobe, a.k, a.batch)
    named = {(100_000, 384, 256, 16, 10, 32): "configs[0]",
             (1_000_000, 768, 1024, 32, 10, 256): "configs[1]",
             (10_000_000, 768, 8192, 32, 10, 256): "configs[3] shape on one GPU"}
    tag = named.get(shape, "custom")
    n = f"{a.n / 1e6:g}M" if a.n >= 1_000_000 else f"{a.n // 1000}K"
    s = (f"{tag}: {n} x {a.d} fp32 IVF per GPU (nlist {a.nlist} per GPU), nprobe {a.nprobe}, "
         f"k {a.k}, {a.batch} queries per GPU per step")
    if world > 1:
        s += (f"; {world} x {n} x {a.d} global index, nlist {world * a.nlist}, lists sharded by "
              "rank (configs[3] shape)")
    return s


# ---------------------------------------------------------------- workload
def make_base(n, d, seed):
    """Unit-sphere fp32 rows (bench/workload.py:108-111 semantics), PCG64."""
    rng = np.random.default_rng(np.random.PCG64(seed))
    out = np.empty((n, d), dtype=np.float32)
    step = 1 << 17
    for i in range(0, n, step):
        x = rng.standard_normal(size=(min(step, n - i), d), dtype=np.float32)
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        out[i:i + len(x)] = x
    return out


def make_queries(base, count, seed):
    """Half perturbed base rows (x + 0.01 N(0, I)), half fresh unit vectors."""
    rng = np.random.default_rng(np.random.PCG64(seed + 7919))
    n, d = base.shape
    q = np.empty((count, d), dtype=np.float32)
    h = count // 2
    q[:h] = base[rng.integers(0, n, h)] + 0.01 * rng.standard_normal(size=(h, d), dtype=np.float32)
    x = rng.standard_normal(size=(count - h, d), dtype=np.float32)
    q[h:] = x / np.linalg.norm(x, axis=1, keepdims=True)
    perm = rng.permutation(count)
    return np.ascontiguousarray(q[perm])


def seed_rows(n, nlist, seed):
    rng = np.random.default_rng(np.random.PCG64(seed + 104729))
    return np.sort(rng.choice(n, nlist, replace=False))


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


def load_traffic():
    p = os.path.join(ROOT, "profiles", "scan_ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
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


def oracle_time(flat, Q, nprobe, k, threads):
    t0 = time.perf_counter()
    res = flat.search(Q, nprobe, k, threads=threads)
    return time.perf_counter() - t0, res


# ---------------------------------------------------------------- reference arm
def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # rank 0 alone runs the CPU arm
    from oracle import oracle as O

    t_build = time.perf_counter()
    base = make_base(a.n, a.d, a.seed)
    seeds = base[seed_rows(a.n, a.nlist, a.seed)].astype(np.float32)
    lab = None
    cents = seeds
    for _ in range(max(1, a.kmeans_iters)):
        lab = np.empty(a.n, dtype=np.int64)
        cn = (cents * cents).sum(1)
        for i in range(0, a.n, 65536):
            blk = base[i:i + 65536]
            lab[i:i + len(blk)] = np.argmin(cn[None, :] - 2.0 * (blk @ cents.T), axis=1)
        cents = np.stack([base[lab == c].mean(0) if np.any(lab == c) else seeds[c]
                          for c in range(a.nlist)]).astype(np.float32)
    order = np.argsort(lab, kind="stable")
    lens = np.bincount(lab, minlength=a.nlist).astype(np.int64)
    off = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    rows = np.ascontiguousarray(base[order])
    ids = order.astype(np.int64)
    live = np.where(lens > 0)[0]
    cent_exact = np.stack([O.centroid(rows[off[c]:off[c] + lens[c]]) for c in live])
    flat = O.FlatIVF(rows, ids, off[live], lens[live], cent_exact, live.astype(np.int64))
    build_s = time.perf_counter() - t_build
    threads = os.cpu_count() or 1
    Qall = make_queries(base, (a.warmup + a.steps) * a.batch, a.seed)
    # size each step's sample so the run stays within ~a minute
    probe_t, _ = oracle_time(flat, Qall[:threads], a.nprobe, a.k, threads)
    per_q = probe_t / threads
    sample = max(1, min(a.batch, int(60.0 / max(1, a.steps) / max(per_q, 1e-6))))
    if a.cpu_sample:
        sample = a.cpu_sample
    for w in range(a.warmup):
        oracle_time(flat, Qall[w * a.batch: w * a.batch + sample], a.nprobe, a.k, threads)
    t_total = 0.0
    for s in range(a.steps):
        lo = (a.warmup + s) * a.batch
        dt, _ = oracle_time(flat, Qall[lo: lo + sample], a.nprobe, a.k, threads)
        t_total += dt
    qps = a.steps * sample / t_total
    line = {
        "impl": "reference", "metric": METRIC, "value": qps, "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1000.0 * t_total / a.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": workload_name(a),
                   "n": a.n, "d": a.d, "nlist": a.nlist, "nprobe": a.nprobe, "k": a.k,
                   "batch": a.batch, "sample_queries_per_step": sample},
        "cpu_baseline": {"value": qps, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{sample} of each step's {a.batch} queries, C oracle "
                                   f"(oracle/pancake_oracle.c) on {threads} threads"},
        "e2e": {"value": qps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "build_s": build_s,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def build_shard(a, rank, dev):
    """This rank's 1M x 768 shard: unit-sphere rows, device k-means (kmeans_assign
    arithmetic, a.kmeans_iters rounds), rows sorted by list.  Returns device
    rows/ids sorted by list, list lengths and offsets, and the host base."""
    import torch

    from paper_2602_21477_b200 import _native as N

    base = make_base(a.n, a.d, a.seed + rank)  # rank r owns shard r (weak scaling)
    X = torch.from_numpy(base).to(dev)
    seeds = X[torch.from_numpy(seed_rows(a.n, a.nlist, a.seed + rank)).to(dev)].contiguous()
    cents = seeds
    labels = torch.empty(a.n, dtype=torch.int64, device=dev)
    dists = torch.empty(a.n, dtype=torch.float64, device=dev)
    for _ in range(max(1, a.kmeans_iters)):
        torch.cuda.synchronize()
        N.check(N.lib().pk_kmeans_assign(X.data_ptr(), a.n, cents.data_ptr(), a.nlist, a.d,
                                         labels.data_ptr(), dists.data_ptr(), N.PK_DEVICE_PTRS))
        sums = torch.zeros(a.nlist, a.d, dtype=torch.float64, device=dev)
        for i in range(0, a.n, 1 << 20):  # fp64 sums in row chunks (10M x 768 would need 61 GB)
            sums.index_add_(0, labels[i:i + (1 << 20)], X[i:i + (1 << 20)].double())
        cnt = torch.bincount(labels, minlength=a.nlist).clamp(min=1).double()
        cents = (sums / cnt[:, None]).float().contiguous()
    order = torch.argsort(labels, stable=True)
    lens = torch.bincount(labels, minlength=a.nlist).cpu().numpy().astype(np.int64)
    del labels, dists
    Xs = X[order].contiguous()
    del X
    ids_sorted = (order + rank * a.n).contiguous()
    torch.cuda.empty_cache()  # the index arena is cudaMalloc'd outside torch's cache
    offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    torch.cuda.synchronize()
    return base, Xs, ids_sorted, lens, offs


def run_ours(a):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PK_BENCH_SHARE_GPU=1: every rank on cuda:0 over gloo -- only to exercise
    # the multi-rank code path on a one-GPU box; never a bench number
    share = os.environ.get("PK_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2602_21477_b200 import DeviceIndex
    from paper_2602_21477_b200 import build as B
    from paper_2602_21477_b200 import _native as N
    from paper_2602_21477_b200.sharded import ShardedIndex, block_offsets

    if rank == 0:
        B.build()
    if dist:
        dist.barrier()
    N.load()

    t_build = time.perf_counter()
    dev = torch.device("cuda", local)
    base, Xs, ids_sorted, lens, offs = build_shard(a, rank, dev)
    reserve = dict(reserve_rows=int(a.n * 1.26) + 32 * a.nlist + 4096, reserve_lists=a.nlist * world)
    sh = None
    if world == 1:
        ix = DeviceIndex(a.d, 0, local, **reserve)
        live = [c for c in range(a.nlist) if lens[c] > 0]
        cent_tab = {c: ix.create_list(c, 0, Xs[offs[c]:offs[c] + lens[c]],
                                      ids_sorted[offs[c]:offs[c] + lens[c]]) for c in live}
    else:
        # global list table: rank r's k-means list c is cid r * nlist + c, owned by r
        lens_all = torch.empty(world * a.nlist, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(lens_all, torch.from_numpy(lens).to(dev))
        lens_all = lens_all.cpu().numpy().reshape(world, a.nlist)
        gl = [(r, c) for r in range(world) for c in range(a.nlist) if lens_all[r, c] > 0]
        gcids = [r * a.nlist + c for r, c in gl]
        sh = ShardedIndex(a.d, 0, local, **reserve)
        ix = sh.local

        def fetch(i):
            c = gl[i][1]
            return Xs[offs[c]:offs[c] + lens[c]], ids_sorted[offs[c]:offs[c] + lens[c]]

        sh.load(gcids, [0] * len(gl), [int(lens_all[r, c]) for r, c in gl], fetch,
                owners=[r for r, _ in gl])
        live = [c for c in range(a.nlist) if lens[c] > 0]
        cent_tab = None
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t_build

    # every rank brings its own batches (perturbed rows of its shard + fresh unit vectors)
    Qall_h = make_queries(base, (a.warmup + a.steps) * a.batch, a.seed + 1000 * rank)
    Qall = torch.from_numpy(Qall_h).to(dev).view(a.warmup + a.steps, a.batch, a.d)
    codes = torch.zeros(1, dtype=torch.int32, device=dev)
    kk = a.k
    o_ids = torch.empty(a.batch, kk, dtype=torch.int64, device=dev)
    o_d = torch.empty(a.batch, kk, dtype=torch.float32, device=dev)
    o_c = torch.empty(a.batch, kk, dtype=torch.int64, device=dev)
    o_n = torch.empty(a.batch, dtype=torch.int32, device=dev)
    o_s = torch.empty(a.batch, dtype=torch.int64, device=dev)
    stream = torch.cuda.ExternalStream(ix.stream_handle(), device=dev)
    bufs = None
    if sh is not None:
        bb = block_offsets(a.batch, kk)["total"]
        bufs = {"probe": torch.empty(a.batch, a.nprobe, dtype=torch.int32, device=dev),
                "q_all": torch.empty(world * a.batch, a.d, dtype=torch.float32, device=dev),
                "probe_all": torch.empty(world * a.batch, a.nprobe, dtype=torch.int32, device=dev),
                "send": torch.empty(world * bb, dtype=torch.uint8, device=dev),
                "recv": torch.empty(world * bb, dtype=torch.uint8, device=dev)}

    # N>1 combine: results written straight into their origin rank's HBM over
    # NVLink (CUDA IPC + device flags, PK_COMBINE=peer, default) or an NCCL
    # all-to-all (PK_COMBINE=nccl, or when the peer mapping cannot be set up)
    combine = None
    if sh is not None:
        combine = os.environ.get("PK_COMBINE", "peer")
        if combine == "peer":
            ok = 1
            try:
                sh.setup_peer_combine(a.batch, kk)
            except Exception as exc:  # no P2P mapping between these devices
                print(f"rank {rank}: peer combine unavailable ({exc})", file=sys.stderr)
                ok = 0
            # every rank must take the same combine path
            flag = torch.tensor([ok], dtype=torch.int32, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 0:
                combine = "nccl"

    def step(s):
        if sh is None:
            ix.search_device(Qall[s], codes, a.nprobe, kk, o_ids, o_d, o_c, o_n, o_s)
        else:
            with torch.cuda.stream(stream):
                if combine == "peer":
                    sh.search_dispatch_peer(Qall[s], codes, a.nprobe, kk, bufs, o_ids, o_d, o_c,
                                            o_n, o_s)
                else:
                    sh.search_dispatch_device(Qall[s], codes, a.nprobe, kk, bufs, o_ids, o_d, o_c,
                                              o_n, o_s)

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
    ms = ev0.elapsed_time(ev1)
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
    if combine == "peer" and ix.combine_status() != 0:
        raise RuntimeError("peer combine timed out waiting for a rank's results")
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_q = world * a.steps * a.batch  # every rank serves its own batch each step
    qps = total_q / (ms / 1000.0)

    # ---- roofline of the fused scan: algorithmic bytes of the distinct local
    # lists each scan launch reads (the probe sets of the same batches)
    row_bytes = 4 * a.d + 8
    alg_bytes = []
    for s in range(a.steps):
        if sh is None:
            out = ix.search(Qall_h[(a.warmup + s) * a.batch:(a.warmup + s + 1) * a.batch], [0],
                            a.nprobe, kk, want_probe=True)
            pr = np.unique(out.probe[out.probe >= 0])
            alg_bytes.append(float(lens[pr].sum()) * row_bytes)
        else:
            step(a.warmup + s)
            torch.cuda.synchronize()
            pa = bufs["probe_all"].cpu().numpy()
            pr = np.unique(pa[pa >= 0])  # list handles = global registration order
            gl_lens = np.array([int(lens_all[r, c]) for r, c in gl], dtype=np.int64)
            mine = np.array([r == rank for r, _ in gl])
            alg_bytes.append(float(gl_lens[pr][mine[pr]].sum()) * row_bytes)
    pool = None
    try:
        if sh is None:
            ix.search(Qall_h[a.warmup * a.batch:(a.warmup + 1) * a.batch], [0], a.nprobe, kk)
        B_last = a.batch * world
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
    traffic = load_traffic()

    # ---- e2e through the public API with host buffers (pinned queries in,
    # results out, every step)
    e2e = None
    if not a.no_e2e:
        Qpin = torch.from_numpy(Qall_h).pin_memory().numpy().reshape(a.warmup + a.steps, a.batch, a.d)

        def host_run(first, count):
            """count host batches: N=1 pipelines two in flight (submit batch
            s+1, then collect batch s: its H2D and the host work overlap the
            device pass of batch s); N>1 runs the dispatch/combine host path."""
            if sh is not None:
                for s in range(first, first + count):
                    sh.search_dispatch(Qpin[s], [0], a.nprobe, kk)
                return
            prev = None
            for s in range(first, first + count):
                t = ix.search_submit(Qpin[s], [0], a.nprobe, kk)
                if prev is not None:
                    ix.search_collect(prev)
                prev = t
            ix.search_collect(prev)

        host_run(0, min(a.warmup, 3))
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        host_run(a.warmup, a.steps)
        e2e_s = time.perf_counter() - t0
        if dist:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": total_q / e2e_s, "unit": UNIT, "h2d_bytes_per_step": a.batch * a.d * 4,
               "d2h_bytes_per_step": a.batch * (kk * (8 + 4 + 8) + 4 + 8),
               "path": ("DeviceIndex.search_submit / search_collect (pk_search_submit / "
                        "pk_search_collect C-ABI, two batches in flight: batch s+1 submitted "
                        "before batch s is collected)" if sh is None else
                        "ShardedIndex.search_dispatch (pk_search_coarse / NCCL / "
                        "pk_search_probed / pk_merge_shards)")
               + ", pinned host query buffer, every step's results read back to host"}

    # ---- CPU baseline (oracle port) + parity on the same sample, rank 0 at N=1
    cpu = parity = None
    if rank == 0 and world == 1:
        from oracle import oracle as O

        threads = os.cpu_count() or 1
        rows_h = Xs.cpu().numpy()
        ids_h = ids_sorted.cpu().numpy()
        cids_l = np.array(live, dtype=np.int64)
        flat = O.FlatIVF(rows_h, ids_h, offs[live], lens[live],
                         np.stack([cent_tab[c] for c in live]), cids_l)
        sample = a.cpu_sample or min(a.batch, max(16, 4 * threads))
        Qs = Qall_h[a.warmup * a.batch: a.warmup * a.batch + sample]
        t_cpu, (r_ids, r_d, r_n, r_p, r_sc) = oracle_time(flat, Qs, a.nprobe, kk, threads)
        cpu = {"value": sample / t_cpu, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"first {sample} queries of timed step 0, C oracle "
                         f"(oracle/pancake_oracle.c), {threads} threads"}
        g = ix.search(Qs, [0], a.nprobe, kk, want_probe=True)
        parity = {"queries": sample,
                  "id_mismatch": int((g.ids != r_ids).sum()),
                  "dist_bit_mismatch": int((g.dists.view(np.uint32) != r_d.view(np.uint32)).sum()),
                  "probe_mismatch": int((g.probe != r_p).sum())}

    if rank == 0:
        per_step = 6 if sh is None else 10  # our kernels per search step
        line = {
            "metric": METRIC, "value": qps, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(a, world),
                       "n_per_gpu": a.n, "d": a.d, "nlist_per_gpu": a.nlist, "nprobe": a.nprobe,
                       "k": a.k, "batch_per_gpu": a.batch,
                       "l2": (f"inputs larger than L2 (index {a.n * (4 * a.d + 8) / 1e9:.2f} GB per "
                              "GPU vs 126 MB L2; each batch reads most lists)"),
                       "parallelism": f"list-sharded x{world}" + (
                           ", dispatch (NCCL all-gather of queries + list handles) / combine ("
                           + ("per-shard top-k written into the origin rank's HBM over NVLink P2P, "
                              "device flags, device merge" if combine == "peer" else
                              "NCCL all-to-all of per-shard top-k, device merge") + ")"
                           if world > 1 else "")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
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
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
