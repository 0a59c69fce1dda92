"""The reference's own test suites, run against this package (VERDICT r1 next
#4; "the new build's parity suite should re-run these
reference tests against the native executor / NativeStore").

Two boundaries are exercised, exactly as a user of the reference would switch:

* the Python API -- ``pkg/tests/test_engine.py`` and
  ``pkg/tests/test_acceptance.py`` import ``Store`` / ``StoreConfig`` /
  ``UsageError`` / ``ScopePermissionError`` / ``OperationBatch`` from
  ``agentmem``; here those names are this package's (and the reference bench
  runner drives this package's ``Store``);
* the executor plugin -- ``pkg/tests/test_tiering.py`` and acceptance
  criterion 06 build the reference's own ``ClusterStore`` + ``TierManager``
  around ``SimulatedAccelerator(CostModel())``; here that name constructs this
  package's ``NativeAccelerator`` (HBM lists, device scans, device k-means).

Everything else the tests import (the bench harness and its brute-force
``StreamingOracle``, ``ClusterStore``, ``TierManager``, the graph and FSM
internals some acceptance criteria test directly) stays the reference's --
the checkers and the unchanged host side.

The reference comes from its offline install in ``baseline/_ref`` (git-ignored,
travels to the GPU box; its ``pkg/tests`` copied to
``baseline/_ref/agentmem_tests``), or ``/root/reference/pkg`` where present.
Tests that still fail against the drop-in are listed in ``DEVIATIONS`` with the
reason (strict xfail, so a fix shows up as XPASS) and in DESIGN.md.
"""

from __future__ import annotations

import importlib
import importlib.util
import os
import sys
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

SUITES = ("test_engine", "test_acceptance", "test_tiering", "test_persist")

# reference test -> why the drop-in differs (strict xfail)
DEVIATIONS: dict[str, str] = {}


def _reference_paths():
    for src, tests in ((os.path.join(ROOT, "baseline", "_ref"),
                        os.path.join(ROOT, "baseline", "_ref", "agentmem_tests")),
                       ("/root/reference/pkg/src", "/root/reference/pkg/tests")):
        if os.path.isdir(os.path.join(src, "agentmem")) and os.path.isdir(tests):
            return src, tests
    return None, None


def _load_suites():
    src, tests = _reference_paths()
    if src is None:
        return {}, "reference package not installed (baseline/_ref)"
    try:
        import numba  # noqa: F401  (the reference's kernels)
    except ImportError:
        return {}, "numba missing: the reference package cannot run"
    # numba must not write its cache into the reference tree
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="pk_numba_"))
    for p in (tests, src):
        if p not in sys.path:
            sys.path.insert(0, p)
    ref = importlib.import_module("agentmem")
    for sub in ("core", "engine", "tiering", "clusters", "graph", "fsm", "pool", "cache",
                "persist", "kernels", "bench", "bench.runner", "bench.oracle"):
        importlib.import_module(f"agentmem.{sub}")

    import paper_2602_21477_b200 as pk
    from paper_2602_21477_b200 import engine as pk_engine
    from paper_2602_21477_b200.accelerator import NativeAccelerator

    # the Python API: the names a user imports from agentmem
    for name in ("Store", "StoreConfig", "SearchResult", "UsageError", "ScopePermissionError",
                 "ParseError", "VersionMismatchError"):
        setattr(ref, name, getattr(pk, name))
    for name in ("Store", "StoreConfig", "SearchResult", "SearchStats", "OperationBatch"):
        setattr(ref.engine, name, getattr(pk_engine, name))
    ref.bench.runner.Store = pk.Store
    ref.bench.runner.StoreConfig = pk.StoreConfig
    # the reference's file helpers the tests call directly (read_fvecs) raise
    # the boundary's error types
    for name in ("ParseError", "UsageError", "VersionMismatchError"):
        setattr(ref.persist, name, getattr(pk, name))

    # the executor plugin: the reference TierManager drives the native executor
    def native_executor(model=None):
        return NativeAccelerator(model, error_type=ref.tiering.AcceleratorError)

    ref.tiering.SimulatedAccelerator = native_executor

    mods = {}
    for suite in SUITES:
        path = os.path.join(tests, f"{suite}.py")
        spec = importlib.util.spec_from_file_location(f"refsuite_{suite}", path)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        mods[suite] = mod
    return mods, None


_MODS, _SKIP = _load_suites()


@pytest.fixture
def rng():
    """pkg/tests/conftest.py."""
    return np.random.default_rng(1234)


def _export(mods):
    """Re-export the reference's test classes / functions for collection."""
    out = {}
    for suite, mod in mods.items():
        for name, obj in vars(mod).items():
            if name.startswith("Test") and isinstance(obj, type):
                out[f"{name}_{suite.removeprefix('test_')}"] = type(
                    f"{name}_{suite.removeprefix('test_')}", (obj,), {})
            elif name.startswith("test_") and callable(obj):
                fn = obj
                if name in DEVIATIONS:
                    fn = pytest.mark.xfail(strict=True, reason=DEVIATIONS[name])(fn)
                out[name] = fn
    return out


if _SKIP:
    def test_reference_suites_unavailable():
        pytest.skip(_SKIP)
else:
    globals().update(_export(_MODS))


def test_suites_loaded_against_this_package():
    """The shim really swapped the boundary (not the reference's own Store)."""
    if _SKIP:
        pytest.skip(_SKIP)
    import agentmem

    import paper_2602_21477_b200 as pk

    assert agentmem.Store is pk.Store
    eng = _MODS["test_engine"]
    assert eng.Store is pk.Store and eng.UsageError is pk.UsageError
    acc = _MODS["test_tiering"].SimulatedAccelerator()
    assert type(acc).__name__ == "NativeAccelerator"
