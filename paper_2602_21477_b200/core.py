"""Foundational value types, mirroring the reference's ``agentmem.core``
(ref/core.py:1-138): metrics (smaller distance = closer; inner product is
negated), vector validation and the error classes callers catch.

Distances are never computed here -- ``batch_distances`` and friends route to
the sm_100a kernels (``kernels.py``).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

STATIC_SCOPE = "static"


class UsageError(ValueError):
    """Caller violated an operation precondition (ref/core.py:20-21)."""


class ScopePermissionError(UsageError):
    """Write attempted on a scope the agent may not modify (ref/core.py:24-25)."""


class ParseError(ValueError):
    """Malformed input file; carries the byte offset (ref/core.py:28-33)."""

    def __init__(self, message: str, offset: int):
        super().__init__(f"{message} (at byte offset {offset})")
        self.offset = offset


class VersionMismatchError(ValueError):
    """Exchange file written by an incompatible format version (ref/core.py:36-37)."""


class AcceleratorError(RuntimeError):
    """Device-side failure (ref/tiering.py:29-30).  The reference falls back to
    the host on this error; this implementation has no host compute path and
    raises it to the caller instead."""


class Metric(Enum):
    SQUARED_EUCLIDEAN = "sq_l2"
    INNER_PRODUCT = "ip"
    COSINE = "cosine"

    @property
    def wire_code(self) -> int:
        return _WIRE_CODES[self]

    @classmethod
    def from_wire(cls, code: int) -> "Metric":
        for m, c in _WIRE_CODES.items():
            if c == code:
                return m
        raise ParseError(f"unknown metric code {code}", 0)


_WIRE_CODES = {
    Metric.SQUARED_EUCLIDEAN: 0,
    Metric.INNER_PRODUCT: 1,
    Metric.COSINE: 2,
}


@dataclass(frozen=True)
class MemoryItem:
    id: int
    vector: np.ndarray
    payload: bytes
    scope: str


def as_vector(values, dimension: int | None = None) -> np.ndarray:
    """Contiguous float32 1-d vector; rejects NaN/Inf and wrong length
    (ref/core.py:74-86)."""
    v = np.ascontiguousarray(values, dtype=np.float32)
    if v.ndim != 1:
        raise UsageError(f"expected a 1-d vector, got shape {v.shape}")
    if dimension is not None and v.shape[0] != dimension:
        raise UsageError(f"dimension mismatch: expected {dimension}, got {v.shape[0]}")
    if not np.all(np.isfinite(v)):
        raise UsageError("vector contains NaN or Inf")
    return v


def as_matrix(values, dimension: int) -> np.ndarray:
    """Batched ``as_vector``: [n, dimension] float32 with the same checks."""
    m = np.ascontiguousarray(values, dtype=np.float32)
    if m.ndim == 1:
        m = m.reshape(1, -1)
    if m.ndim != 2:
        raise UsageError(f"expected a 2-d batch, got shape {m.shape}")
    if m.shape[1] != dimension:
        raise UsageError(f"dimension mismatch: expected {dimension}, got {m.shape[1]}")
    if not np.all(np.isfinite(m)):
        raise UsageError("vector contains NaN or Inf")
    return m


def is_agent_scope(scope: str) -> bool:
    return scope != STATIC_SCOPE


# Device-backed numerics re-exported under the reference names.
from .kernels import batch_distances, centroid, deviation, distance  # noqa: E402,F401
