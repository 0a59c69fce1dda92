"""The reference's coarse graph at its DEFAULT ef (VERDICT r1
missing #3): HybridGraphIndex.search / search_independent (ref/graph.py:
321-422) are approximate best-first traversals, so which lists a query probes
depends on the graph's exact shape.  The Store builds that graph as the
reference does (levels and portal coins from the shared stream, neighbor
lists from device-computed distances) and searches it on the device
(pk_graph.cu).  Traces recorded from the reference at ef_search_factor 4 / 2
-- multi-scope agent graphs grown by k-means splits, portals, hybrid and
per-agent coarse modes, inserts / deletes / updates -- must replay bit-exact,
including SearchStats.coarse_computations (the traversal's distance count)."""

import numpy as np
import pytest

from replay import compare_records, gen, load_golden, replay_store

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", list(gen.GRAPH_TRACE_SPECS))
def test_default_ef_trace_matches_reference(name):
    want = load_golden(f"trace_{name}.npz")
    got = replay_store(gen.GRAPH_TRACE_SPECS[name])
    mism = compare_records(got, want)
    assert not mism, "\n".join(mism[:10])
    assert any(k.endswith("/coarse") for k in want)


@pytest.mark.parametrize("name", ["graph_hybrid"])
def test_default_ef_trace_batched_path(name):
    """The same trace through search_batch (one fused device pass per query
    batch: traversal -> scan -> re-rank)."""
    want = load_golden(f"trace_{name}.npz")
    got = replay_store(gen.GRAPH_TRACE_SPECS[name], batch_searches=True)
    mism = compare_records(got, want)
    assert not mism, "\n".join(mism[:10])
