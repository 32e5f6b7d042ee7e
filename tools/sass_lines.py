#!/usr/bin/env python
"""Attribute an ncu SASS source page to CUDA source lines (ncu's own CUDA-source view
needs the source on the profiling box; this joins the per-instruction metrics with
``nvdisasm -g`` line info of the same .so instead).

usage: python tools/sass_lines.py REPORT.ncu-rep KERNEL_REGEX MANGLED_SUBSTR [--so LIB] [--top N]

Prints per (file, line): warp-stall samples, instructions executed (warp level),
share of each, sorted by samples.
"""
from __future__ import annotations

import argparse
import csv
import io
import os
import re
import subprocess
import tempfile
from collections import defaultdict


def line_map(so: str, mangled_sub: str, outer: bool = False) -> list[tuple[str, int]]:
    """Per instruction (in order) of the first function whose name contains
    ``mangled_sub``: the innermost (file, line) nvdisasm attributes it to, or with
    ``outer`` the kernel-level line it is inlined at."""
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, check=True,
                   stdout=subprocess.DEVNULL)
    out = []
    for cub in sorted(os.listdir(tmp)):
        txt = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)], capture_output=True,
                             text=True).stdout
        inside = False
        cur = ("?", 0)
        fresh = True  # first "//## File" line of a group = innermost; the last = outermost
        for ln in txt.splitlines():
            if ln.startswith(".text."):
                if inside:
                    break
                inside = mangled_sub in ln
                continue
            if not inside:
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                if fresh or outer:
                    cur = (os.path.basename(m.group(1)), int(m.group(2)))
                fresh = False
                continue
            if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln):
                out.append(cur)
                fresh = True
        if out:
            return out
    raise SystemExit(f"function containing {mangled_sub!r} not found in {so}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("mangled")
    ap.add_argument("--so", default="paper_1202_6163_b200/libpfresample.so")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--outer", action="store_true", help="attribute inlined code to the kernel-level line")
    a = ap.parse_args()
    csv_txt = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--kernel-name",
                              f"regex:{a.kernel}", "--print-source", "sass"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(csv_txt)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    body = [r for r in rows[hdr_i + 1:] if r and r[0].startswith("0x")]
    i_s, i_e = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    lm = line_map(a.so, a.mangled, a.outer)
    if len(lm) != len(body):
        print(f"warning: {len(lm)} instructions in the .so vs {len(body)} in the report")
    agg = defaultdict(lambda: [0, 0])
    for k, r in enumerate(body):
        key = lm[k] if k < len(lm) else ("?", 0)
        agg[key][0] += int(float(r[i_s] or 0))
        agg[key][1] += int(float(r[i_e] or 0))
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print(f"total samples {ts}, warp instructions {ti}")
    print("| file:line | samples | share | warp inst | share |")
    print("|---|---|---|---|---|")
    for (f, l), (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:a.top]:
        print(f"| {f}:{l} | {s} | {s / ts:.3f} | {e} | {e / ti:.3f} |")


if __name__ == "__main__":
    main()
