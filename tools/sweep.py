#!/usr/bin/env python
"""Throughput sweep over P and weight variance (BASELINE metric "resampled particles/sec
vs P and weight variance"; SURVEY §8(d) companion sweep P = 2^4 ... 2^24).

Single filters (N = 1) and batches with N * P = 2^26 (P <= 2^16), every scheme,
sigma^2 in {0.1, 1, 10}; R calls captured in a CUDA graph and replayed, timed
with CUDA events (device time per call; inputs resident in HBM).  JSON lines.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def time_calls(fn, reps, dev):
    """Device time per call: the calls are captured in a CUDA graph (so Python / launch
    overhead is not on the timeline) and replayed; warm-up on the capture stream."""
    import torch

    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(3):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) / (3 * reps)


def write_md(rows, path):
    """Markdown tables (particles/s) from the JSON rows of main()."""
    schemes = []
    for r in rows:
        if r["scheme"] not in schemes:
            schemes.append(r["scheme"])
    out = ["# Round 1 sweep: resample-only throughput vs P and weight variance (tools/sweep.py)", "",
           "One B200, device time per call of `pf_resample_batched` (calls captured in a CUDA graph; inputs "
           "resident in HBM). Single filters (N = 1) and batches with N x P = 2^26. Values are particles/s. "
           "Raw: `profiles/r01_sweep.jsonl`.", ""]
    for batched in (False, True):
        out += ["## " + ("batches (N x P = 2^26)" if batched else "single filter (N = 1)"), "",
                "| P | sigma^2 | " + " | ".join(schemes) + " |", "|---|---|" + "---|" * len(schemes)]
        cells = {}
        for r in rows:
            if r["batched"] == batched:
                cells[(r["P"], r["var"], r["scheme"])] = r["particles_per_s"]
        for P, var in sorted({(k[0], k[1]) for k in cells}):
            lp = P.bit_length() - 1
            vals = [f"{cells.get((P, var, sc), float('nan')):.2e}" for sc in schemes]
            out.append(f"| 2^{lp} | {var} | " + " | ".join(vals) + " |")
        out.append("")
    with open(path, "w") as f:
        f.write("\n".join(out) + "\n")


def main():
    import torch

    import paper_1202_6163_b200 as pf
    import pfinputs

    dev = torch.device("cuda:0")
    md = sys.argv[sys.argv.index("--md") + 1] if "--md" in sys.argv else None
    rows = []
    cases = [("systematic", 0, 0), ("stratified", 0, 0), ("multinomial", 0, 0),
             ("multinomial", 0, pf.PF_SORTED), ("metropolis", 32, 0)]
    for batched in (False, True):
        for lp in range(4, 25, 2):
            P = 1 << lp
            if batched and P > (1 << 16):
                continue
            N = (1 << 26) // P if batched else 1
            for var in (0.1, 1.0, 10.0):
                x = pfinputs.gaussian_logw_torch(P, var, pfinputs.BASE_SEED + lp, N, dev)
                anc = torch.empty((N, P), dtype=torch.int32, device=dev)
                for scheme, B, flags in cases:
                    reps = 20 if N * P <= (1 << 22) else 5
                    ms = time_calls(lambda: pf.pf_resample_batched(scheme, x, 5, B=B, ancestors=anc, flags=flags),
                                    reps, dev)
                    name = scheme + ("_sorted_a6" if flags else "") + (f"_B{B}" if B else "")
                    row = {"batched": batched, "N": N, "P": P, "var": var, "scheme": name,
                           "us_per_call": round(ms * 1e3, 2), "particles_per_s": N * P / (ms / 1e3)}
                    rows.append(row)
                    print(json.dumps(row))
                    sys.stdout.flush()
    if md:
        write_md(rows, md)


if __name__ == "__main__":
    main()
