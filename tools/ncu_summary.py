#!/usr/bin/env python
"""Summarise an ncu report (``--set full``) into a markdown table for profiles/.

usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--alg name=bytes ...] > profiles/rNN_x.md

Per kernel: duration, DRAM read/write bytes (the roofline ``traffic``), DRAM
throughput % of peak, L2 / L1 throughput, issue-active %, warps-active %,
registers, occupancy limiter, and the top three stall reasons.
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys

KEYS = {
    "dur": "gpu__time_duration.sum",
    "rd": "dram__bytes_read.sum",
    "wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "occ_regs": "launch__occupancy_limit_registers",
    "occ_smem": "launch__occupancy_limit_shared_mem",
    "grid": "launch__grid_size",
}
STALL_PREFIX = "smsp__average_warps_issue_stalled_"
STALL_SUFFIX = "_per_issue_active.ratio"

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "s": 1e3}


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def val(hdr, units, row, key, to=None):
    if key not in hdr:
        return None
    i = hdr.index(key)
    s = row[i].replace(",", "")
    try:
        v = float(s)
    except ValueError:
        return row[i]
    u = units[i]
    if to == "bytes":
        v *= SCALE.get(u, 1)
    elif to == "ms":
        v *= SCALE.get(u, 1)
    return v


def short(name):
    name = name.replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    return name.split("(")[0].strip()[:48]


def main():
    rep = sys.argv[1]
    hdr, units, rows = load(rep)
    stall_keys = [h for h in hdr if h.startswith(STALL_PREFIX) and h.endswith(STALL_SUFFIX)]
    print(f"ncu report `{rep}` ({len(rows)} kernel launches)\n")
    print("| kernel | ms | DRAM rd GB | DRAM wr GB | DRAM % | L2 % | L1 % | issue % | warps % | regs | occ lim (reg/smem) | grid | top stalls (warps per issue) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        name = short(r[hdr.index("Kernel Name")])
        dur = val(hdr, units, r, KEYS["dur"], "ms")
        rd = val(hdr, units, r, KEYS["rd"], "bytes")
        wr = val(hdr, units, r, KEYS["wr"], "bytes")
        stalls = []
        for k in stall_keys:
            v = val(hdr, units, r, k)
            if isinstance(v, float):
                stalls.append((v, k[len(STALL_PREFIX):-len(STALL_SUFFIX)]))
        stalls.sort(reverse=True)
        top = ", ".join(f"{n} {v:.2f}" for v, n in stalls[:3])

        def f(key, fmt="{:.1f}"):
            v = val(hdr, units, r, KEYS[key])
            return fmt.format(v) if isinstance(v, float) else str(v)

        print(f"| {name} | {dur:.4f} | {rd / 1e9:.3f} | {wr / 1e9:.3f} | {f('dram_pct')} | {f('l2_pct')} | "
              f"{f('l1_pct')} | {f('issue')} | {f('warps')} | {f('regs', '{:.0f}')} | "
              f"{f('occ_regs', '{:.0f}')}/{f('occ_smem', '{:.0f}')} | {f('grid', '{:.0f}')} | {top} |")


if __name__ == "__main__":
    main()
