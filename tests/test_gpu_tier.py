"""The native cold tier (ref/tiering.py:175-448):
lists live in pinned host memory, HBM holds the hotset, probed cold lists are
streamed into HBM staging, admissions copy on a side stream.  Residency must
never change a result (ref/tiering.py:294-328): every check below is
bit-exact against the oracle / the reference fixtures."""

import numpy as np
import pytest

from oracle import oracle as O
from replay import compare_records, gen, load_golden, replay_store

pytestmark = pytest.mark.gpu


def bits(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


def _check(ix, lists, cents, cids, Q, nprobe, kk):
    flat = O.FlatIVF.from_lists(lists, np.stack(cents), np.asarray(cids, np.int64))
    out = ix.search(Q, [0], nprobe, kk, want_probe=True)
    ids, dd, cnt, probe, sc = flat.search(Q, nprobe, kk, threads=8)
    assert np.array_equal(out.probe, probe)
    assert np.array_equal(out.ids, ids)
    assert np.array_equal(bits(out.dists), bits(dd))
    assert np.array_equal(out.scanned, sc)


@pytest.mark.parametrize("stage", ["gather", "dma"])
def test_tiered_index_every_residency_state(stage, monkeypatch):
    """Both staging paths: the zero-copy gather kernel (default) and the copy
    engines (PK_STAGE=dma: one DMA per contiguous run of lists, ids and norms
    by a kernel)."""
    from paper_2602_21477_b200 import DeviceIndex

    monkeypatch.setenv("PK_STAGE", stage)

    rng = np.random.default_rng(21)
    d, nlist = 96, 30
    ix = DeviceIndex(d)
    ix.enable_tier()
    centers = rng.normal(size=(nlist, d)).astype(np.float32)
    lists, cents, cids, nid = [], [], [], 0
    for c in range(nlist):
        n = int(rng.integers(1, 900))
        rows = (centers[c] + 0.5 * rng.normal(size=(n, d))).astype(np.float32)
        ids = rng.permutation(np.arange(nid, nid + n)).astype(np.int64)
        nid += n
        cents.append(ix.create_list(c + 7, 0, rows, ids))
        lists.append([ids, rows])
        cids.append(c + 7)
        assert ix.residency(c + 7) == 0  # created cold
        assert np.array_equal(bits(cents[-1]), bits(O.centroid(rows)))
    Q = (centers[rng.integers(0, nlist, 90)] + 0.5 * rng.normal(size=(90, d))).astype(np.float32)
    _check(ix, [tuple(x) for x in lists], cents, cids, Q, 6, 10)  # all cold: staged
    st = ix.tier_stats()
    assert st["cold_lists"] == nlist and st["staged_lists_last"] > 0
    # admit a third; search immediately (copies may be in flight) and again
    for c in cids[::3]:
        ix.set_resident(c, True)
    _check(ix, [tuple(x) for x in lists], cents, cids, Q, 6, 10)
    ix.sync()
    _check(ix, [tuple(x) for x in lists], cents, cids, Q, 9, 20)
    assert all(ix.residency(c) == 1 for c in cids[::3])
    # mutations on resident, cold and in-flight lists, then evictions
    for j, c in enumerate(cids[:8]):
        if j == 5:
            ix.set_resident(c, True)  # in flight while appended to
        add = rng.normal(size=(300, d)).astype(np.float32)
        aid = np.arange(nid, nid + 300)
        nid += 300
        ix.append(c, add, aid)
        lists[j][0] = np.concatenate([lists[j][0], aid])
        lists[j][1] = np.concatenate([lists[j][1], add])
        for _ in range(7):
            r = int(rng.integers(0, len(lists[j][0])))
            ix.remove_row(c, r)
            last = len(lists[j][0]) - 1
            lists[j][0][r] = lists[j][0][last]
            lists[j][1][r] = lists[j][1][last]
            lists[j][0] = lists[j][0][:last]
            lists[j][1] = lists[j][1][:last]
        cents[j] = ix.recompute(c)
        assert np.array_equal(bits(cents[j]), bits(O.centroid(lists[j][1])))
        rows, ids = ix.read(c)
        assert np.array_equal(ids, lists[j][0]) and np.array_equal(bits(rows), bits(lists[j][1]))
    _check(ix, [tuple(x) for x in lists], cents, cids, Q, 6, 10)
    for c in cids[::3]:
        ix.set_resident(c, False)
    ix.set_resident(cids[1], True)
    _check(ix, [tuple(x) for x in lists], cents, cids, Q, 30, 64)
    st = ix.tier_stats()
    assert st["admissions_started"] >= 11 and st["staged_bytes_total"] > 0
    ix.close()


@pytest.mark.parametrize("name,budget", [("ivf_small", 40_000), ("ivf_splits", 8_000)])
def test_store_trace_with_native_cold_tier(name, budget):
    """The reference's recorded traces (inserts, deletes, updates, centroid
    maintenance, k-means splits, multi-scope searches) replayed on a Store
    whose budget keeps only part of the index in HBM, with the hotset policy
    running every 3 operations: identical results, real residency churn."""
    want = load_golden(f"trace_{name}.npz")
    log = []
    got = replay_store(gen.TRACE_SPECS[name], overrides=dict(accelerator="native", budget_bytes=budget,
                                                              hotset_interval=3), tier_log=log)
    mism = compare_records(got, want)
    assert not mism, "\n".join(mism[:10])
    assert any(m["tier_cold_lists"] > 0 for m in log), "budget never left a list cold"
    assert any(m["tier_resident_lists"] > 0 for m in log), "hotset never admitted a list"
    assert max(m["tier_staged_searches"] for m in log) > 0


@pytest.mark.parametrize("mode", ["host", "device", "async"])
def test_staging_ranges_recycled(mode):
    """Every tiered batch stages its probed cold lists into HBM arena ranges;
    those ranges go back to the arena after the batch (they used to
    leak, so the arena grew by the staged bytes on every search).  Over many
    batches -- host-pointer, device-pointer and async searches, with host-arena
    mutations (appends, swap-with-last removals) between them -- the arena's
    high-water mark stays bounded and every result stays exact."""
    import torch

    from paper_2602_21477_b200 import DeviceIndex

    rng = np.random.default_rng(5)
    d, nlist = 64, 40
    ix = DeviceIndex(d)
    ix.enable_tier()
    centers = rng.normal(size=(nlist, d)).astype(np.float32)
    lists, cents, cids, nid = [], [], [], 0
    for c in range(nlist):
        n = int(rng.integers(50, 700))
        rows = (centers[c] + 0.5 * rng.normal(size=(n, d))).astype(np.float32)
        ids = np.arange(nid, nid + n, dtype=np.int64)
        nid += n
        cents.append(ix.create_list(c, 0, rows, ids))
        lists.append([ids, rows])
        cids.append(c)
    for c in cids[::4]:
        ix.set_resident(c, True)
    ix.sync()
    total_rows = sum(len(x[0]) for x in lists)
    tops = []
    dev = torch.device("cuda", 0)
    for it in range(40):
        Q = (centers[rng.integers(0, nlist, 32)] + 0.5 * rng.normal(size=(32, d))).astype(np.float32)
        nprobe = int(rng.integers(3, 12))
        if mode == "host":
            out = ix.search(Q, [0], nprobe, 10)
            ids_g = out.ids
        elif mode == "device":
            Qd = torch.from_numpy(Q).to(dev)
            codes = torch.zeros(1, dtype=torch.int32, device=dev)
            o_ids = torch.empty(32, 10, dtype=torch.int64, device=dev)
            o_d = torch.empty(32, 10, dtype=torch.float32, device=dev)
            o_c = torch.empty(32, 10, dtype=torch.int64, device=dev)
            o_n = torch.empty(32, dtype=torch.int32, device=dev)
            o_s = torch.empty(32, dtype=torch.int64, device=dev)
            ix.search_device(Qd, codes, nprobe, 10, o_ids, o_d, o_c, o_n, o_s)
            ix.sync()
            ids_g = o_ids.cpu().numpy()
        else:
            t = ix.search_submit(Q, [0], nprobe, 10)
            ids_g = ix.search_collect(t).ids
        flat = O.FlatIVF.from_lists([tuple(x) for x in lists], np.stack(cents),
                                    np.asarray(cids, np.int64))
        r_ids = flat.search(Q, nprobe, 10, threads=8)[0]
        assert np.array_equal(ids_g, r_ids), f"batch {it}"
        # host-arena mutations between batches (the last gather may be in flight)
        j = int(rng.integers(0, nlist))
        add = (centers[j] + 0.5 * rng.normal(size=(5, d))).astype(np.float32)
        aid = np.arange(nid, nid + 5, dtype=np.int64)
        nid += 5
        ix.append(cids[j], add, aid)
        lists[j][0] = np.concatenate([lists[j][0], aid])
        lists[j][1] = np.concatenate([lists[j][1], add])
        r = int(rng.integers(0, len(lists[j][0])))
        ix.remove_row(cids[j], r)
        last = len(lists[j][0]) - 1
        lists[j][0][r] = lists[j][0][last]
        lists[j][1][r] = lists[j][1][last]
        lists[j][0] = lists[j][0][:last]
        lists[j][1] = lists[j][1][:last]
        cents[j] = ix.recompute(cids[j])
        tops.append(ix.tier_stats()["arena_top_rows"])
    # resident quarter (+25% slack) plus at most ~two batches of staging
    assert max(tops) < 3 * total_rows, tops
    assert max(tops[20:]) <= 1.5 * max(tops[:20]), tops
    ix.close()


def test_native_admission_abort_and_flush_count():
    """The native tier's counterparts of the reference's fault seam and flush
    criterion (ref/tiering.py:280-290, 357-361, 404-416; pkg/tests
    test_acceptance.py:256-266): an injected admission-allocation failure
    aborts the admission -- the cluster stays cold with all of its items and
    searches stay exact -- and the next hotset pass admits it; inserts into a
    resident cluster count a flush exactly at every b_insert-th insert."""
    from paper_2602_21477_b200 import Store, StoreConfig

    rng = np.random.default_rng(9)
    d = 16
    store = Store(StoreConfig(dimension=d, accelerator="native", budget_bytes=1 << 30,
                              cache_enabled=False, splits_enabled=False, hotset_interval=1 << 30))
    base = rng.normal(size=(400, d)).astype(np.float32)
    store.load_lists("static", [(np.arange(i * 100, (i + 1) * 100), base[i * 100:(i + 1) * 100])
                                for i in range(4)])
    tier = store.tier
    for c in store.clusters.clusters:
        tier.record_access(c)
    tier.fail_next_alloc = True
    tier.hotset_update()  # first admission aborts, the other three go in
    assert tier.aborted == 1 and not tier.fail_next_alloc
    cold = [c for c, cl in store.clusters.clusters.items() if cl.resident is None]
    assert len(cold) == 1
    assert store.index.residency(cold[0]) == 0 and store.clusters.clusters[cold[0]].size == 100
    q = rng.normal(size=d).astype(np.float32)
    res = store.search(None, ["static"], q, 10, 4)
    dd = O.distances(q, base)
    want = np.lexsort((np.arange(400), dd))[:10]
    assert res.ids == want.tolist()
    assert np.array_equal(bits(res.distances), bits(dd[want]))
    tier.hotset_update()  # retried: admitted now
    assert all(cl.resident is not None for cl in store.clusters.clusters.values())
    assert tier.metrics()["aborted_admissions"] == 1
    # flush equivalent: every b_insert-th insert into a resident list
    target = next(iter(store.clusters.clusters))
    cent = store.clusters.clusters[target].centroid
    assert tier.flush_count == 0
    for i in range(1, tier.b_insert + 1):
        v = (cent + 1e-3 * rng.normal(size=d)).astype(np.float32)
        store.insert(None, "static", [v])
        assert tier.flush_count == (1 if i >= tier.b_insert else 0), i
    store.close()
