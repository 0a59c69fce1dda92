"""Agent mode (SURVEY.md 8a rows a9-a11, configs[2]): per-agent multi-level
caches, staged inserts merged down into base clusters, early termination,
FSM pattern hints, prefetch, profiles and verify mode, replayed against
traces recorded from the reference Store (tests/golden/make_golden.py
--agents).  Bit-exact: hits, distances, scopes, scanned counts, scan_ids,
level reached, early-termination flags, final clusters, staged sets and
cache statistics."""

import numpy as np
import pytest

from replay import compare_records, gen, load_golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", list(gen.AGENT_TRACE_SPECS))
def test_agent_trace_search_batches(name):
    """The same traces with each run of an agent's searches submitted as one
    search_batch: the queries are answered one by one (each one's side
    effects shape the next), their coarse traversals and probed-list rows
    come from ONE device pass (pk_agent_lists) while the lists are unchanged."""
    from paper_2602_21477_b200 import Store, StoreConfig
    from paper_2602_21477_b200.core import Metric
    from paper_2602_21477_b200.pnck import write_pnck

    spec = gen.AGENT_TRACE_SPECS[name]
    want = load_golden(f"agent_{name}.npz")
    base, ops = gen.agent_trace_ops(spec)
    store = Store(StoreConfig(**gen.agent_store_config_kwargs(spec)))
    calls = [0, 0]  # batched passes, searches answered from one
    lists_fn, pf_fn = store.index.agent_lists, store._prefetched_lists

    def counted_lists(*a, **kw):
        calls[0] += 1
        return lists_fn(*a, **kw)

    def counted_pf(*a, **kw):
        out = pf_fn(*a, **kw)
        calls[1] += out is not None
        return out

    store.index.agent_lists = counted_lists
    store._prefetched_lists = counted_pf
    got = gen.run_agent_ops(store, spec, base, ops, write_pnck, Metric(spec.get("metric", "sq_l2")),
                            group_searches=True)
    mism = compare_records(got, want)
    assert not mism, "\n".join(mism[:10])
    assert calls[0] > 0 and calls[1] > 0, calls
    store.close()


@pytest.mark.parametrize("name", list(gen.AGENT_TRACE_SPECS))
def test_agent_trace_matches_reference(name):
    from paper_2602_21477_b200 import Store, StoreConfig
    from paper_2602_21477_b200.core import Metric
    from paper_2602_21477_b200.pnck import write_pnck

    spec = gen.AGENT_TRACE_SPECS[name]
    want = load_golden(f"agent_{name}.npz")
    base, ops = gen.agent_trace_ops(spec)
    store = Store(StoreConfig(**gen.agent_store_config_kwargs(spec)))
    got = gen.run_agent_ops(store, spec, base, ops, write_pnck, Metric(spec.get("metric", "sq_l2")))
    mism = compare_records(got, want)
    assert not mism, "\n".join(mism[:10])
    early = sum(1 for k in want if k.endswith("/early") and bool(want[k]))
    assert early > 10, "the trace must exercise early termination"
    if spec["verify"]:
        assert sum(int(want[f"final/agent{a}/verified"]) for a in range(spec["n_agents"])) > 0
    store.close()


@pytest.mark.parametrize("seed", range(6))
def test_most_similar_pattern_pair_equals_pairwise_loop(seed):
    """observe_completed's pattern-table merge choice from one device matrix
    over every pattern's states equals the reference's pairwise loop of
    fsm_pair_similarity (ref/fsm.py:372-378), ties included."""
    from paper_2602_21477_b200.core import Metric
    from paper_2602_21477_b200.fsm import (AccessPatternFsm, FsmState, _most_similar_pair,
                                           fsm_pair_similarity)

    rng = np.random.default_rng(seed)
    d = 32
    base = rng.normal(size=(6, d)).astype(np.float32)
    fsms = []
    for _ in range(int(rng.integers(3, 18))):
        n = int(rng.integers(1, 9))
        # shared rows make exact ties between pairs
        c = [base[int(rng.integers(0, 6))] if rng.random() < 0.4 else rng.normal(size=d).astype(np.float32)
             for _ in range(n)]
        fsms.append(AccessPatternFsm([FsmState(v, 0.1, 1, 1) for v in c], {}, [0] * n, 0.1))
    best = (0, 1, -1.0)
    for i in range(len(fsms) - 1):
        for j in range(i + 1, len(fsms)):
            s = fsm_pair_similarity(fsms[i], fsms[j], Metric.SQUARED_EUCLIDEAN)
            if s > best[2]:
                best = (i, j, s)
    assert _most_similar_pair(fsms, Metric.SQUARED_EUCLIDEAN) == best[:2]
