"""Snapshot / restore (ref/persist.py:136-380) -- SURVEY.md section 8f #3,
VERDICT r1 b1 / f3.

The snapshot is the reference's file format, so besides the reference's own
persistence tests (tests/test_gpu_reference_suite.py runs pkg/tests/
test_persist.py and acceptance criterion 09 against this package) a snapshot
moves between the two packages: written here and restored by the reference
(and the other way round), both restored stores then run the same probes and
the same agent traffic, with bit-identical answers, cache levels and
early-termination flags.  The reference side runs in a subprocess from its
offline install (baseline/_ref)."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import persist_recipe as R

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _has_reference():
    return any(os.path.isdir(os.path.join(p, "agentmem"))
               for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"))


def _ref(mode, path, tmp_path):
    out = tmp_path / f"ref_{mode}.json"
    subprocess.run([sys.executable, os.path.join(ROOT, "tests", "persist_recipe.py"), mode, str(path),
                    str(out)], check=True, timeout=900)
    return json.loads(out.read_text())


@pytest.fixture
def ours():
    from paper_2602_21477_b200 import Store, StoreConfig

    return Store, StoreConfig


def test_round_trip_probes_and_counters(ours, tmp_path):
    Store, StoreConfig = ours
    s = R.build(Store, StoreConfig)
    p = tmp_path / "s.pnck"
    s.snapshot(p)
    r = Store.restore(p)
    # a restored store snapshots to the same bytes (before any further op)
    p2 = tmp_path / "s2.pnck"
    r.snapshot(p2)
    assert p2.read_bytes() == p.read_bytes()
    assert r._next_item_id == s._next_item_id and r.live_count() == s.live_count()
    assert r.caches["a1"].d_agent == s.caches["a1"].d_agent
    for iid in list(s.clusters.owner)[:20]:
        assert r.get_item(iid)[1] == s.get_item(iid)[1]
    assert r.rng.bit_generator.state == s.rng.bit_generator.state
    assert R.probes(r) == R.probes(s)
    s.close()
    r.close()


def test_snapshot_bit_exact_across_runs(ours, tmp_path):
    Store, StoreConfig = ours
    pa, pb = tmp_path / "a.pnck", tmp_path / "b.pnck"
    a, b = R.build(Store, StoreConfig), R.build(Store, StoreConfig)
    a.snapshot(pa)
    b.snapshot(pb)
    assert pa.read_bytes() == pb.read_bytes()


@pytest.mark.skipif(not _has_reference(), reason="reference package not installed (baseline/_ref)")
def test_same_ops_same_snapshot_as_the_reference(ours, tmp_path):
    """The same op sequence on both packages writes byte-identical snapshots:
    every cluster row and centroid, graph, pattern table, cache pool, counter
    and the RNG state agree."""
    Store, StoreConfig = ours
    ref_path = tmp_path / "ref.pnck"
    ref = _ref("build", ref_path, tmp_path)
    s = R.build(Store, StoreConfig)
    p = tmp_path / "ours.pnck"
    s.snapshot(p)
    assert R.probes(s) == ref["probes"]
    from paper_2602_21477_b200 import pnck

    _, _, rec_a, sec_a = pnck.read_pnck(p, with_sections=True)
    _, _, rec_b, sec_b = pnck.read_pnck(ref_path, with_sections=True)
    assert len(rec_a) == len(rec_b)
    for (ca, ia, ma), (cb, ib, mb) in zip(rec_a, rec_b):
        assert np.array_equal(ia, ib) and np.array_equal(ma.view(np.uint32), mb.view(np.uint32))
        assert np.array_equal(ca.view(np.uint32), cb.view(np.uint32))
    assert sorted(sec_a) == sorted(sec_b)
    for tag in sec_a:
        assert json.loads(sec_a[tag]) == json.loads(sec_b[tag]), tag
    assert p.read_bytes() == ref_path.read_bytes()


@pytest.mark.skipif(not _has_reference(), reason="reference package not installed (baseline/_ref)")
def test_our_snapshot_restored_by_the_reference(ours, tmp_path):
    Store, StoreConfig = ours
    s = R.build(Store, StoreConfig)
    p = tmp_path / "ours.pnck"
    s.snapshot(p)
    ref = _ref("restore", p, tmp_path)
    r = Store.restore(p)
    assert R.probes(r) == ref["probes"]
    assert R.continuation(r) == ref["continuation"]


@pytest.mark.skipif(not _has_reference(), reason="reference package not installed (baseline/_ref)")
def test_reference_snapshot_restored_here(ours, tmp_path):
    Store, StoreConfig = ours
    p = tmp_path / "ref.pnck"
    _ref("build", p, tmp_path)
    ref = _ref("restore", p, tmp_path)
    r = Store.restore(p)
    assert R.probes(r) == ref["probes"]
    assert R.continuation(r) == ref["continuation"]
