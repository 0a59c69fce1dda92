"""Host-side logic that needs no GPU: config validation, PNCK exchange format,
scope interning, locking, the graph-RNG mirror, shard planning."""

import os
import struct
import threading

import numpy as np
import pytest

from paper_2602_21477_b200 import Metric, ParseError, StoreConfig, UsageError, VersionMismatchError
from paper_2602_21477_b200.clusters import CoarseRngMirror
from paper_2602_21477_b200.concurrency import RWLock, TaskRunner
from paper_2602_21477_b200.engine import OperationBatch, ScopeCodes, profile_promote, profile_reorder
from paper_2602_21477_b200.pnck import read_pnck, write_pnck


class TestConfig:
    def test_defaults_match_reference(self):
        c = StoreConfig(dimension=8)
        assert (c.split_threshold, c.split_target, c.maintenance_interval) == (4096, 2048, 256)
        assert (c.kappa, c.alpha_et, c.b_insert, c.default_nprobe) == (2, 0.7, 128, 8)
        assert c.metric is Metric.SQUARED_EUCLIDEAN

    @pytest.mark.parametrize("kw", [dict(dimension=0), dict(dimension=4, alpha_et=1.5),
                                    dict(dimension=4, split_target=10, split_threshold=10),
                                    dict(dimension=4, coarse_mode="x"), dict(dimension=4, accelerator="gpu")])
    def test_invalid(self, kw):
        with pytest.raises(UsageError):
            StoreConfig(**kw)

    def test_metric_string(self):
        assert StoreConfig(dimension=3, metric="cosine").metric is Metric.COSINE

    def test_batch_kind(self):
        with pytest.raises(UsageError):
            OperationBatch("frobnicate", None, [])


class TestPnck:
    def test_round_trip(self, tmp_path):
        rng = np.random.default_rng(0)
        d = 5
        cl = [(rng.normal(size=d).astype(np.float32), np.array([3, 1, 2 ** 40]),
               rng.normal(size=(3, d)).astype(np.float32)),
              (np.zeros(d, np.float32), np.array([], dtype=np.int64), np.zeros((0, d), np.float32))]
        p = tmp_path / "x.pnck"
        write_pnck(p, d, Metric.COSINE, cl, sections=[(b"META", b"{}")])
        dim, metric, recs = read_pnck(p)
        assert dim == d and metric is Metric.COSINE and len(recs) == 2
        assert recs[0][1].tolist() == [3, 1, 2 ** 40]
        assert np.array_equal(recs[0][2], cl[0][2]) and np.array_equal(recs[0][0], cl[0][0])
        assert len(recs[1][1]) == 0
        # the snapshot's tagged sections come back in order (persist.restore)
        write_pnck(p, d, Metric.COSINE, cl, sections=[(b"CMET", b'{"a":1}'), (b"META", b"")])
        *_, secs = read_pnck(p, with_sections=True)
        assert list(secs) == [b"CMET", b"META"] and secs[b"CMET"] == b'{"a":1}' and secs[b"META"] == b""
        p.write_bytes(p.read_bytes() + b"TAG")  # truncated section
        with pytest.raises(ParseError):
            read_pnck(p, with_sections=True)

    def test_snapshot_config_fields_are_the_references(self):
        """CONF carries exactly the reference's StoreConfig fields, so the
        reference's StoreConfig(**conf) accepts our snapshots."""
        import dataclasses

        from paper_2602_21477_b200.engine import StoreConfig
        from paper_2602_21477_b200.persist import REFERENCE_CONFIG_FIELDS

        ours = [f.name for f in dataclasses.fields(StoreConfig)]
        assert [f for f in ours if f not in REFERENCE_CONFIG_FIELDS] == ["device", "sharded"]
        assert all(f in ours for f in REFERENCE_CONFIG_FIELDS)

    def test_layout_bytes(self, tmp_path):
        """Byte layout of ref/persist.py:66-94."""
        p = tmp_path / "y.pnck"
        write_pnck(p, 2, Metric.SQUARED_EUCLIDEAN, [(np.array([1, 2], np.float32), np.array([7]),
                                                     np.array([[3, 4]], np.float32))])
        b = open(p, "rb").read()
        want = b"PNCK" + struct.pack("<IIB", 1, 2, 0) + struct.pack("<I", 1)
        want += struct.pack("<2f", 1, 2) + struct.pack("<I", 1) + struct.pack("<Q", 7) + struct.pack("<2f", 3, 4)
        assert b == want

    def test_errors(self, tmp_path):
        p = tmp_path / "z.pnck"
        p.write_bytes(b"NOPE")
        with pytest.raises(ParseError):
            read_pnck(p)
        p.write_bytes(b"PNCK" + struct.pack("<IIB", 2, 4, 0))
        with pytest.raises(VersionMismatchError):
            read_pnck(p)
        p.write_bytes(b"PNCK" + struct.pack("<IIB", 1, 4, 0) + struct.pack("<I", 1) + b"\0" * 10)
        with pytest.raises(ParseError):
            read_pnck(p)


def test_scope_codes():
    s = ScopeCodes()
    assert s.intern("static") == 0 and s.intern("a") == 1 and s.intern("static") == 0
    assert s.mask_codes(["a", "static"]).tolist() == [0, 1]


def test_profiles():
    assert profile_reorder([3, 1, 9], [0, 1, 2, 3]) == [3, 1, 0, 2]
    assert profile_promote([1, 2, 3], [3, 5, 3], 3) == [3, 5, 1]


def test_profile_order_equals_reorder():
    """The vectorised scan order equals profile_reorder over range(size)."""
    from paper_2602_21477_b200.engine import profile_order, profile_reorder

    rng = np.random.default_rng(4)
    cases = [([], 5), ([3, 1, 3, 0], 4), ([9, 2, -1, 2], 3), ([0], 0), ([7, 7], 8)]
    cases += [(rng.integers(-3, 40, int(rng.integers(0, 30))).tolist(), int(rng.integers(0, 40)))
              for _ in range(200)]
    for entries, size in cases:
        want = profile_reorder(entries, list(range(size)))
        assert profile_order(entries, size).tolist() == want


@pytest.mark.parametrize("ordered", [True, False])
def test_vector_pool_matches_list_model(ordered):
    """VectorPool (head offset for FIFO pops, swap-with-last for unordered
    pools) keeps the reference's row order (ref/pool.py:33-144)."""
    from paper_2602_21477_b200.pool import VectorPool

    from paper_2602_21477_b200.rowstore import RowStore

    rng = np.random.default_rng(11 if ordered else 12)
    d = 5
    store = RowStore(None, d)  # slots only: the uploads are checked, not sent
    pool = VectorPool(d, ordered=ordered, rows=store)
    model = []  # [(id, vec, scope, staged)] in scan order
    dev = {}  # what the device row store would hold: slot -> row
    nid = 0
    for step in range(3000):
        op = rng.integers(0, 5)
        if op == 4 and model:
            # promote_many: remove (staged |= prior) + add per item, in order
            items = []
            for j in rng.permutation(len(model))[:int(rng.integers(1, 5))].tolist():
                iid, v = model[j][0], model[j][1]
                if rng.integers(0, 4) == 0:
                    v = rng.normal(size=d).astype(np.float32)  # a changed vector: re-uploaded
                items.append((iid, v, int(rng.integers(0, 3)), bool(rng.integers(0, 2))))
            for _ in range(int(rng.integers(0, 3))):
                items.append((nid, rng.normal(size=d).astype(np.float32), int(rng.integers(0, 3)),
                              bool(rng.integers(0, 2))))
                nid += 1
            pool.promote_many(items)
            for iid, v, sc, st in items:
                at = [m[0] for m in model].index(iid) if iid in [m[0] for m in model] else None
                if at is not None:
                    st = st or model[at][3]
                    if ordered:
                        model.pop(at)
                    else:
                        last = model.pop()
                        if at < len(model):
                            model[at] = last
                model.append((iid, v, sc, st))
        elif op <= 1 or not model:
            v = rng.normal(size=d).astype(np.float32)
            sc, st = int(rng.integers(0, 3)), bool(rng.integers(0, 2))
            assert pool.add(nid, v, sc, st)
            model.append((nid, v, sc, st))
            nid += 1
        elif op == 2:
            j = int(rng.integers(0, len(model)))
            iid = model[j][0]
            assert pool.remove(iid)
            if ordered:
                model.pop(j)
            else:
                last = model.pop()
                if j < len(model):
                    model[j] = last
        else:
            if ordered:
                got = pool.pop_front()
                want = model.pop(0)
                assert got[0] == want[0] and np.array_equal(got[1], want[1]) and got[2:] == want[2:]
            else:
                iid = model[0][0]
                pool.set_staged(iid, True)
                model[0] = model[0][:3] + (True,)
        assert len(pool) == len(model)
        assert pool.ids.tolist() == [m[0] for m in model]
        if model:
            assert np.array_equal(pool.vectors, np.stack([m[1] for m in model]))
            assert pool.scopes.tolist() == [m[2] for m in model]
            j = int(rng.integers(0, len(model)))
            assert pool.row_of(model[j][0]) == j
            assert pool.staged_flag(model[j][0]) == model[j][3]
            assert [r[0] for r in pool.rows()] == [m[0] for m in model]
            assert pool.scope_mask([1]).tolist() == [m[2] == 1 for m in model]
            lut = np.zeros(4, dtype=bool)
            lut[1] = True
            ids, sl = pool.in_scope(lut, (1,))
            assert ids.tolist() == [m[0] for m in model if m[2] == 1]
        # every live row's slot is distinct, and after applying the queued
        # uploads the slot holds exactly that row (freed slots never leak)
        ps, pr = store.take_puts()
        if ps is not None:
            for s_, r_ in zip(ps.tolist(), pr):
                dev[s_] = r_
        slots = pool.slots.tolist()
        assert len(set(slots)) == len(slots) and min(slots, default=0) >= 0
        assert store.live == len(model)
        for s_, m in zip(slots, model):
            assert np.array_equal(dev[s_], m[1])


def test_running_kth_equals_kth_smallest():
    """The incremental stop-rule statistic equals ref/cache.py:154-160's k-th
    smallest of the concatenation after every chunk (duplicates counted)."""
    from paper_2602_21477_b200.cache import RunningKth, kth_smallest

    rng = np.random.default_rng(0)
    for _ in range(500):
        k = int(rng.integers(1, 30))
        run, chunks = RunningKth(k), []
        for _ in range(int(rng.integers(1, 8))):
            c = rng.integers(0, 20, int(rng.integers(0, 40))).astype(np.float32)
            chunks.append(c)
            run.add(c)
            assert run.kth() == kth_smallest(chunks, k)


def test_rwlock_and_runner():
    lock = RWLock()
    hits = []

    def reader():
        with lock.read():
            hits.append(1)

    ts = [threading.Thread(target=reader) for _ in range(4)]
    with lock.write():
        for t in ts:
            t.start()
    for t in ts:
        t.join()
    assert len(hits) == 4
    r = TaskRunner(0)
    assert r.submit("search", lambda x: x + 1, 1).result() == 2
    r2 = TaskRunner(4)
    assert r2.submit("update", lambda: 5).result() == 5
    r2.shutdown()


def test_coarse_rng_mirror_matches_model():
    """Same draws as the oracle store model's graph-insert restatement."""
    from oracle.store_model import StoreModel

    m = StoreModel(4, seed=9)
    m.register("a")
    rng = np.random.default_rng(np.random.PCG64(9))
    mirror = CoarseRngMirror(rng)
    mirror.register_scope("static")
    mirror.register_scope("a")
    for scope in ["static", "a", "static", "a", "a", "static"]:
        m._graph_insert(scope)
        mirror.on_insert(scope)
    assert m.rng.random() == rng.random()


class _FakeCluster:
    def __init__(self, cid, n, d=8):
        self.id, self.size, self.dimension = cid, n, d
        self.member_ids = np.arange(n, dtype=np.int64)
        self.resident = None
        self.buffer = []

    @property
    def nbytes(self):
        return self.size * self.dimension * 4


class _FakeIndex:
    def __init__(self):
        self.res = {}

    def set_resident(self, cid, on):
        self.res[cid] = bool(on)


class _FakeStore:
    def __init__(self):
        self.clusters = {}


def _tier(budget):
    from paper_2602_21477_b200.tiering import TierManager

    st, ix = _FakeStore(), _FakeIndex()
    return st, ix, TierManager(st, ix, budget_bytes=budget, native=True)


class TestHotsetPolicy:
    """The native tier's policy is the reference's TierManager.hotset_update
    (ref/tiering.py:222-262); these mirror ref tests/test_tiering.py:51-104."""

    def test_zero_budget_empty(self):
        st, ix, tier = _tier(0)
        st.clusters[0] = _FakeCluster(0, 1)
        tier.record_access(0)
        tier.hotset_update()
        assert tier.hotset == set() and ix.res == {}

    def test_single_cluster_admitted(self):
        st, ix, tier = _tier(1 << 30)
        st.clusters[0] = _FakeCluster(0, 1)
        tier.record_access(0)
        assert tier.hotset_update() == [("admit", 0)]
        assert tier.hotset == {0} and ix.res == {0: True}
        assert st.clusters[0].resident is not None

    def test_budget_invariant(self):
        st, ix, tier = _tier(10 * 8 * 4 * 3)  # room for three 10-vector clusters
        for g in range(6):
            st.clusters[g] = _FakeCluster(g, 10)
            for _ in range(g + 1):
                tier.record_access(g)
        tier.hotset_update()
        assert sum(st.clusters[c].nbytes for c in tier.hotset) <= tier.budget_bytes
        assert tier.hotset == {5, 4, 3}  # hottest first, greedy under the budget

    def test_vectorised_update_equals_the_loop(self):
        """hotset_update ranks and fills the budget with arrays; the target
        set equals the reference loop's (sorted by (-freq, cid), greedy
        under the budget, skipping empty / never-accessed clusters) over
        random sizes, access streams, ties and budgets."""
        rng = np.random.default_rng(5)
        for trial in range(40):
            n = int(rng.integers(1, 60))
            budget = int(rng.integers(0, 8 * 4 * 40 * n // 3 + 2))
            st, ix, tier = _tier(budget)
            for g in range(n):
                st.clusters[g] = _FakeCluster(g, int(rng.integers(0, 40)))
            for _ in range(int(rng.integers(0, 4 * n))):
                tier.record_access(int(rng.integers(0, n)))
            if trial % 3 == 0:  # exact ties: same counts, same recency pattern
                for g in range(n):
                    tier.freq[g] = (1.0, tier.clock)
            clusters = st.clusters
            live = [c for c in clusters if clusters[c].size > 0]
            freq = {c: tier.decayed_freq(c) for c in live}
            want, used = set(), 0
            for cid in sorted(live, key=lambda c: (-freq[c], c)):
                nb = clusters[cid].nbytes
                if nb == 0 or freq[cid] <= 0.0:
                    continue
                if used + nb <= budget:
                    want.add(cid)
                    used += nb
            tier.hotset_update()
            assert tier.hotset == want

    def test_hysteresis_and_eviction(self):
        st, ix, tier = _tier(8 * 4 * 10)  # room for one 10-vector cluster
        st.clusters[0] = _FakeCluster(0, 10)
        st.clusters[1] = _FakeCluster(1, 10)
        for _ in range(10):
            tier.record_access(0)
        tier.hotset_update()
        assert tier.hotset == {0}
        for _ in range(11):  # 1 is hotter, but not by the 1.2 hysteresis factor:
            tier.record_access(1)  # 0 is retained next to it (ref/tiering.py:244-252)
        assert tier.hotset_update() == [("admit", 1)]
        assert tier.hotset == {0, 1}
        for _ in range(20):
            tier.record_access(1)  # no new displacer: 0 falls out of the target
        assert tier.hotset_update() == [("evict", 0)]
        assert tier.hotset == {1} and ix.res == {0: False, 1: True}

    def test_zipf_hit_rate_near_offline_oracle(self):
        rng = np.random.default_rng(0)
        st, ix, tier = _tier(8 * 8 * 4 * 100)
        for i in range(1000):
            st.clusters[i] = _FakeCluster(i, 1, 8)
        zipf = 1.0 / np.arange(1, 1001)
        zipf /= zipf.sum()
        trace = rng.choice(1000, size=20000, p=zipf)
        hits = 0
        for t, cid in enumerate(trace.tolist()):
            hits += cid in tier.hotset
            tier.record_access(cid)
            if t % 200 == 0:
                tier.hotset_update()
        counts = np.bincount(trace, minlength=1000)
        oracle = counts[np.argsort(-counts)[:100]].sum()
        assert hits / len(trace) >= oracle / len(trace) - 0.05


def test_stop_rule_by_count_equals_kth():
    """The agent path's stop rule, kth_smallest(scanned, k) < thresh
    (ref/cache.py:154-160, 199-203; ref/engine.py:391-396), is evaluated as
    "at least k scanned distances are below thresh" (cache.replay and the L2
    list loop): the same decision for every prefix, NaNs and ties included."""
    from paper_2602_21477_b200.cache import kth_smallest

    rng = np.random.default_rng(5)
    for trial in range(400):
        k = int(rng.integers(1, 12))
        chunks = []
        for _ in range(int(rng.integers(1, 9))):
            c = rng.integers(0, 6, size=int(rng.integers(0, 7))).astype(np.float32) / 2
            if rng.random() < 0.2 and len(c):
                c[rng.integers(0, len(c))] = np.nan
            chunks.append(c)
        thresh = float(rng.integers(0, 7)) / 2 if rng.random() < 0.9 else float("nan")
        below = 0
        for j in range(len(chunks)):
            kth = kth_smallest([c for c in chunks[:j + 1] if len(c)], k) if any(len(c) for c in chunks[:j + 1]) else None
            want = kth is not None and kth < thresh
            below += int(np.count_nonzero(chunks[j] < thresh))
            assert (below >= k) == want, (trial, j)


def test_batched_adds_equal_sequential():
    """VectorPool.add_many / L1Cluster.add_many (the capture's batched adds)
    leave the same rows, slots' uploads and bit-identical fp64 running sums as
    add() one item at a time (ref/cache.py:44-51)."""
    from paper_2602_21477_b200.cache import L1Cluster
    from paper_2602_21477_b200.rowstore import RowStore

    rng = np.random.default_rng(3)
    d = 37
    for trial in range(20):
        sa, sb = RowStore(None, d), RowStore(None, d)
        a, b = L1Cluster(d, sa), L1Cluster(d, sb)
        base = [(int(i), (rng.normal(size=d) * 10 ** rng.uniform(-3, 3)).astype(np.float32),
                 int(rng.integers(0, 3)), bool(rng.integers(0, 2))) for i in range(int(rng.integers(0, 9)))]
        for it in base:
            a.add(*it)
            b.add(*it)
        new = [(100 + i, (rng.normal(size=d) * 10 ** rng.uniform(-3, 3)).astype(np.float32),
                int(rng.integers(0, 3)), bool(rng.integers(0, 2))) for i in range(int(rng.integers(1, 25)))]
        for it in new:
            a.add(*it)
        b.add_many(new)
        assert a._sum.tobytes() == b._sum.tobytes()
        assert a.centroid.tobytes() == b.centroid.tobytes()
        assert a.pool.ids.tolist() == b.pool.ids.tolist()
        assert np.array_equal(a.pool.vectors, b.pool.vectors)
        assert a.pool.scopes.tolist() == b.pool.scopes.tolist()
        assert [a.pool.staged_flag(i) for i in a.pool.ids] == [b.pool.staged_flag(i) for i in b.pool.ids]
        pa, pb = sa.take_puts(), sb.take_puts()
        assert sorted(pa[0].tolist()) == sorted(pb[0].tolist())


def test_topk_big_part_equals_chunks():
    """Store._topk with the probed lists' rows passed as one view (``big``)
    returns exactly what the chunked call returns: ties at the cut, ids
    duplicated across chunks, deleted ids (no owner) and the expansion past
    4k + 16 candidates included."""
    from types import SimpleNamespace

    from paper_2602_21477_b200.engine import Store

    rng = np.random.default_rng(11)
    for trial in range(200):
        n_big, n_small = int(rng.integers(0, 400)), int(rng.integers(0, 60))
        pool = int(rng.integers(5, 300))
        bi = rng.integers(0, pool, n_big).astype(np.int64)
        bd = rng.integers(0, 40, n_big).astype(np.float32) / 8  # many exact ties
        si = rng.integers(0, pool, n_small).astype(np.int64)
        sd = rng.integers(0, 40, n_small).astype(np.float32) / 8
        owner = {i: ("cluster", 0) for i in range(pool) if rng.random() < 0.7}
        fake = SimpleNamespace(clusters=SimpleNamespace(owner=owner, clusters={0: SimpleNamespace(scope="s")}))
        k = int(rng.integers(1, 25))
        small = [si[:n_small // 2], si[n_small // 2:]]
        smalld = [sd[:n_small // 2], sd[n_small // 2:]]
        want = Store._topk(fake, [bi[:n_big // 3], bi[n_big // 3:]] + small,
                           [bd[:n_big // 3], bd[n_big // 3:]] + smalld, k)
        got = Store._topk(fake, small, smalld, k, (bi, bd))
        assert got == want, trial


def test_stop_rule_segment_counts():
    """The read phase's per-list below-threshold counts (segmented sum with a
    sentinel, empty lists 0) equal the prefix-count formulation."""
    rng = np.random.default_rng(12)
    for _ in range(300):
        lens = rng.integers(0, 6, int(rng.integers(1, 12)))
        lens[rng.random(len(lens)) < 0.3] = 0
        pre = np.concatenate(([0], np.cumsum(lens)))
        all_d = rng.random(int(pre[-1])).astype(np.float32)
        thresh = float(rng.random())
        nsel = int(rng.integers(1, len(lens) + 1))
        m2 = np.zeros(int(pre[nsel]) + 1, dtype=bool)
        np.less(all_d[:pre[nsel]], thresh, out=m2[:-1])
        cnt = np.add.reduceat(m2, pre[:nsel], dtype=np.int64)
        cnt[pre[:nsel] == pre[1:nsel + 1]] = 0
        cb = np.concatenate(([0], np.cumsum(all_d < thresh)))
        assert np.array_equal(np.cumsum(cnt), cb[pre[1:nsel + 1]])
