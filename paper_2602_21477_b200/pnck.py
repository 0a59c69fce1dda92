"""PNCK exchange format (ref/persist.py:1-130, 383-424), vectorized.

Layout (little-endian): "PNCK", version u32 = 1, dimension u32, metric u8;
u32 cluster count; per cluster: centroid f32[d], u32 n, n x (u64 id, f32[d]);
then tagged sections {tag[4], u64 length, payload} that cluster importers skip.
The reference reads each member with a struct.unpack loop (29 s for
1M x 768); here each record is one numpy view.
"""

from __future__ import annotations

import struct

import numpy as np

from .core import Metric, ParseError, VersionMismatchError

MAGIC = b"PNCK"
VERSION = 1


def write_pnck(path, dimension: int, metric: Metric, clusters, sections=None):
    """clusters: iterable of (centroid f32[d], ids i64[n], rows f32[n, d])."""
    rec = np.dtype([("id", "<u8"), ("v", "<f4", (dimension,))])
    clusters = list(clusters)
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<IIB", VERSION, dimension, metric.wire_code))
        f.write(struct.pack("<I", len(clusters)))
        for cent, ids, rows in clusters:
            f.write(np.ascontiguousarray(cent, dtype="<f4").reshape(dimension).tobytes())
            ids = np.asarray(ids, dtype=np.int64)
            f.write(struct.pack("<I", len(ids)))
            r = np.empty(len(ids), dtype=rec)
            r["id"] = ids.astype(np.uint64)
            r["v"] = np.asarray(rows, dtype=np.float32).reshape(len(ids), dimension)
            f.write(r.tobytes())
        for tag, payload in (sections or []):
            f.write(tag)
            f.write(struct.pack("<Q", len(payload)))
            f.write(payload)


def read_pnck(path, with_sections: bool = False):
    """Returns (dimension, metric, [(centroid, ids i64, rows f32[n, d])]), plus
    {tag: payload} of the tagged sections when ``with_sections``."""
    with open(path, "rb") as f:
        buf = f.read()
    off = 0

    def take(n, what):
        nonlocal off
        if off + n > len(buf):
            raise ParseError(f"truncated file while reading {what}", off)
        s = buf[off:off + n]
        off += n
        return s

    magic = take(4, "magic")
    if magic != MAGIC:
        raise ParseError(f"bad magic {magic!r}", 0)
    (version,) = struct.unpack("<I", take(4, "version"))
    if version != VERSION:
        raise VersionMismatchError(f"format version {version} not supported (expected {VERSION})")
    (dimension,) = struct.unpack("<I", take(4, "dimension"))
    metric = Metric.from_wire(take(1, "metric")[0])
    (count,) = struct.unpack("<I", take(4, "cluster count"))
    rec = np.dtype([("id", "<u8"), ("v", "<f4", (dimension,))])
    out = []
    for ci in range(count):
        cent = np.frombuffer(take(4 * dimension, f"cluster {ci} centroid"), dtype="<f4").copy()
        (n,) = struct.unpack("<I", take(4, f"cluster {ci} member count"))
        if off + n * rec.itemsize > len(buf):
            raise ParseError(f"truncated file while reading cluster {ci} vector", off)
        r = np.frombuffer(buf, dtype=rec, count=n, offset=off)
        off += n * rec.itemsize
        out.append((cent, r["id"].astype(np.int64), np.ascontiguousarray(r["v"], dtype=np.float32)))
    # tagged sections: validated (and skipped by cluster importers)
    sections = {}
    while off < len(buf):
        if off + 4 > len(buf):
            raise ParseError("truncated section tag", off)
        tag = buf[off:off + 4]
        off += 4
        (length,) = struct.unpack("<Q", take(8, "section length"))
        sections[tag] = take(length, f"section {tag!r}")
    if with_sections:
        return dimension, metric, out, sections
    return dimension, metric, out
