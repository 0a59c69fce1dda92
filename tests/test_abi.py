"""The C-ABI library: loads, exports every symbol include/pancake_b200.h
declares, is built for sm_100a, and its distance loops are free of fused
multiply-adds (the reference rounds every op).  No GPU needed."""

import os
import re
import shutil
import subprocess

import pytest

from paper_2602_21477_b200 import _native
from paper_2602_21477_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pancake_b200.h")


@pytest.fixture(scope="module")
def lib():
    B.build()
    return _native.load()


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(pk_\w+)\(", src, re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "pk_search" in syms and "pk_assign" in syms and "pk_distances" in syms
    assert len(syms) >= 20


def test_library_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), f"{s} missing from libpancake_b200.so"
    assert set(_native.EXPORTED) >= set(declared_symbols())


def test_version_without_device(lib):
    assert lib.pk_version() == 1


def _sass():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump unavailable")
    return subprocess.run([exe, "-sass", B.OUT], check=True, capture_output=True, text=True).stdout


def _functions(sass):
    out, cur = {}, None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            out[cur] = []
        elif cur:
            out[cur].append(line)
    return out


def test_built_for_sm100a(lib):
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump unavailable")
    out = subprocess.run([exe, "-lelf", B.OUT], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_distance_kernels_have_no_fma(lib):
    """sq_l2 / neg_ip scans and dense distances must not contract (FFMA)."""
    funcs = _functions(_sass())
    checked = 0
    for name, lines in funcs.items():
        if ("scan_kernelILi0" in name or "scan_kernelILi1" in name or
                "dist_dense_kernelILi0" in name or "dist_dense_kernelILi1" in name):
            body = "\n".join(lines)
            assert not re.search(r"\bFFMA2?\b", body), f"fused multiply-add in {name}"
            checked += 1
    assert checked >= 12


def test_scan_uses_tma(lib):
    funcs = _functions(_sass())
    scan = [n for n in funcs if "scan_kernel" in n]
    assert scan
    for n in scan:
        body = "\n".join(funcs[n])
        assert "UTMALDG" in body and "UBLKCP" in body, f"{n} lacks TMA tensor/bulk copies"
