#!/usr/bin/env python
"""Kernel evidence for bench.py's roofline `traffic` from one `ncu --set full` report: per
kernel launch, DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) and warp instructions
(smsp__inst_executed.sum), keyed "workload/scheme" -> library trace name (the kernel name up to
its template arguments).  Merges into profiles/kernel_evidence.json.

usage: python tools/evidence.py REPORT.ncu-rep c3/systematic [--source "how it was captured"]"""
from __future__ import annotations

import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "kernel_evidence.json")


def main():
    global OUT
    rep, key = sys.argv[1], sys.argv[2]
    if "--out" in sys.argv:
        OUT = sys.argv[sys.argv.index("--out") + 1]
    src = sys.argv[sys.argv.index("--source") + 1] if "--source" in sys.argv else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    col = {n: i for i, n in enumerate(h)}
    ev = {}
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        full = r[col["Kernel Name"]]
        name = re.sub(r"^.*::", "", re.split(r"[<(]", full)[0].strip())
        name = {"k_bsearch_buckets": "k_bsearch", "k_gather_rows16": "k_gather_inplace",
                "k_metro_fpc": "k_metro", "k_hist_smem": "k_hist", "k_hist_runs": "k_hist"}.get(name, name)
        num = lambda m: float(r[col[m]].replace(",", ""))  # noqa: E731
        dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
        e = {"dram_bytes": int(dram), "warp_inst": int(num("smsp__inst_executed.sum")),
             "ncu_ms": num("gpu__time_duration.sum") / 1e6, "variant": full}
        ev[name] = e  # the last launch (after the warm-up calls)
    data = {}
    if os.path.exists(OUT):
        data = json.load(open(OUT))
    data[key] = ev
    data.setdefault("_source", {})[key] = src
    json.dump(data, open(OUT, "w"), indent=1)
    print(json.dumps({key: ev}, indent=1))


if __name__ == "__main__":
    main()
