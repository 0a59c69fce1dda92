#!/usr/bin/env python3
"""Per-source-line warp-stall samples of one kernel in an ncu report.

ncu's CSV source page is per SASS instruction without line numbers; this maps
instruction i of the kernel to the source line nvdisasm -g attributes to it
(same library build) and sums the samples per line.

    python tools/ncu_lines.py gpurun_out/scan_c0.ncu-rep scan_tc_kernelILi0E \
        [--so paper_2602_21477_b200/libpancake_b200.so] [--top 25]
"""

from __future__ import annotations

import argparse
import csv
import io
import os
import re
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sass_lines(so: str, pattern: str):
    """[(file, line) per instruction] of the first function whose mangled name
    contains `pattern`."""
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=td, check=True,
                       capture_output=True)
        for cub in sorted(f for f in os.listdir(td) if f.endswith(".cubin")):
            txt = subprocess.run(["nvdisasm", "-g", os.path.join(td, cub)], capture_output=True,
                                 text=True).stdout
            out, cur, on = [], None, False
            for ln in txt.splitlines():
                if re.match(r"\s*\.text\.", ln) or ln.startswith(".section") or "\t.text." in ln:
                    pass
                m = re.match(r"\s*\.section\s+\.text\.(\S+),", ln)
                if m:
                    if on:
                        break
                    on = pattern in m.group(1)
                    continue
                if not on:
                    continue
                m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
                if m:
                    cur = (os.path.basename(m.group(1)), int(m.group(2)))
                    continue
                if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln):
                    out.append(cur)
            if out:
                return out
    return []


def main():
    p = argparse.ArgumentParser()
    p.add_argument("report")
    p.add_argument("pattern", help="substring of the kernel's mangled name")
    p.add_argument("--so", default=os.path.join(ROOT, "paper_2602_21477_b200", "libpancake_b200.so"))
    p.add_argument("--top", type=int, default=25)
    a = p.parse_args()
    src = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    data = rows[rows.index(hdr) + 1:]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    lines = sass_lines(a.so, a.pattern)
    if len(lines) != len(data):
        print(f"warning: {len(lines)} SASS instructions from nvdisasm vs {len(data)} in the report")
    agg, why = {}, {}
    for k, r in enumerate(data[:len(lines)]):
        key = lines[k]
        v = int(r[si] or 0)
        agg[key] = agg.get(key, 0) + v
        w = why.setdefault(key, {})
        for c in stall_cols:
            x = int(r[hdr.index(c)] or 0)
            if x:
                w[c[6:]] = w.get(c[6:], 0) + x
    tot = sum(agg.values()) or 1
    srcs = {}
    print(f"{tot} samples, {len(data)} instructions")
    print("| share | samples | file:line | top stalls | source |")
    print("|---|---|---|---|---|")
    for key, v in sorted(agg.items(), key=lambda kv: -kv[1])[:a.top]:
        if key is None:
            continue
        f, ln = key
        if f not in srcs:
            path = next((os.path.join(dp, f) for dp, _, fs in os.walk(os.path.join(ROOT, "paper_2602_21477_b200"))
                         if f in fs), None)
            srcs[f] = open(path).read().splitlines() if path else []
        text = srcs[f][ln - 1].strip() if ln - 1 < len(srcs[f]) else ""
        top = ", ".join(f"{k} {c}" for k, c in sorted(why[key].items(), key=lambda kv: -kv[1])[:2])
        print(f"| {100 * v / tot:.1f}% | {v} | {f}:{ln} | {top} | `{text[:70]}` |")


if __name__ == "__main__":
    main()
