#!/usr/bin/env python3
"""Summarize ncu evidence into profiles/ (tracked): the launch list (per-kernel
mean device time, share of a search step) and, for --set full captures, the
roofline counters, pipe utilisation and top stall reasons.

    python tools/ncu_summary.py gpurun_out/launches.csv gpurun_out/scan_full.ncu-rep ... \
        --out profiles/r01_ncu_summary.md [--traffic-json profiles/scan_ncu_traffic.json]
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
]


def to_bytes(val, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return float(val.replace(",", "")) * mult


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    unit = "ns"
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            name = r[ki].split("(")[0]
            agg[name].append(float(r[vi].replace(",", "")))
            unit = r[ui]
    return agg, unit


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("inputs", nargs="+")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic-json")
    ap.add_argument("--title", default="ncu summary")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    traffic = None
    for inp in a.inputs:
        if inp.endswith(".csv"):
            agg, unit = launches(inp)
            total = sum(sum(v) / len(v) for v in agg.values())
            lines += [f"## Launch list `{inp.split('/')[-1]}` (cold-cache, serialised; compare shares)", "",
                      f"| kernel | launches | mean ({unit}) | share of step |", "|---|---|---|---|"]
            for k, v in sorted(agg.items(), key=lambda t: -sum(t[1]) / len(t[1])):
                m = sum(v) / len(v)
                lines.append(f"| `{k}` | {len(v)} | {m:,.0f} | {100 * m / total:.1f}% |")
            lines.append("")
        else:
            h, units, rows = raw(inp)
            for row in rows:
                name = row[h.index("Kernel Name")] if "Kernel Name" in h else "?"
                lines += [f"## `{inp.split('/')[-1]}`: {name.split('(')[0]}", "", "| metric | value |", "|---|---|"]
                vals = {}
                for k in KEYS:
                    if k in h:
                        i = h.index(k)
                        vals[k] = (row[i], units[i])
                        lines.append(f"| {k} | {row[i]} {units[i]} |")
                stalls = [(h[i], float(row[i].replace(",", "") or 0)) for i in range(len(h))
                          if "pcsamp_warps_issue_stalled" in h[i] and not h[i].endswith("not_issued")]
                tot = sum(v for _, v in stalls) or 1.0
                lines += ["", "Top stall reasons (PC sampling):", ""]
                for k, v in sorted(stalls, key=lambda t: -t[1])[:8]:
                    lines.append(f"- {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {100 * v / tot:.1f}%")
                lines.append("")
                if "scan_kernel" in name and "dram__bytes_read.sum" in vals:
                    rb = to_bytes(*vals["dram__bytes_read.sum"])
                    wb = to_bytes(*vals["dram__bytes_write.sum"])
                    traffic = {"kernel": name.split("(")[0], "dram_bytes_per_launch": rb + wb,
                               "dram_read": rb, "dram_write": wb, "source": inp.split("/")[-1]}
    with open(a.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if a.traffic_json and traffic:
        with open(a.traffic_json, "w") as f:
            json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
