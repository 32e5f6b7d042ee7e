#!/usr/bin/env python
"""Throughput sweep over P and weight variance (BASELINE metric "resampled particles/sec
vs P and weight variance"; SURVEY §8(d) companion sweep P = 2^4 ... 2^24).

Single filters (N = 1) and batches with N * P = 2^26 (P <= 2^16), every scheme,
sigma^2 in {0.1, 1, 10}.  Two timings per case: cold (L2 flushed before every call,
inputs from HBM; fraction of the HBM roofline from the library-stated algorithmic
bytes) and warm (calls replayed back to back in a CUDA graph: working sets below
L2 stay resident; fraction of the measured L2 read bandwidth for those).  JSON lines.
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


def cold_time(fn, reps, dev, scratch):
    """Device time per call with L2 flushed before every call (a 512 MiB scratch write between
    calls, outside the timed interval): the inputs come from HBM, as in a PF loop whose step
    touches more than L2 between two resamplings."""
    import torch

    s = torch.cuda.current_stream(dev)
    for _ in range(2):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for k in range(reps):
        scratch.fill_(k)
        ev[k][0].record(s)
        fn()
        ev[k][1].record(s)
    torch.cuda.synchronize(dev)
    return sum(a.elapsed_time(b) for a, b in ev) / reps


def alg_bytes(pf, fn, dev):
    """Algorithmic HBM bytes of one call as the library states them (sum over its launches)."""
    import torch

    pf.pf_profile_enable(True)
    fn()
    kt = pf.pf_profile_collect()
    pf.pf_profile_enable(False)
    torch.cuda.synchronize(dev)
    return sum(v[2] for v in kt.values()), {k: v[0] for k, v in kt.items()}


def peaks_from_files():
    hbm = 6549.1
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"])
    except Exception:
        pass
    l2 = None
    try:
        with open(os.path.join(ROOT, "profiles", "r02_microbench.jsonl")) as f:
            for line in f:
                d = json.loads(line)
                if d.get("bench") == "l2_stream":
                    l2 = float(d["GBs"])
    except Exception:
        pass
    return hbm, l2


def write_md(rows, path, hbm, l2):
    """Markdown tables from the JSON rows of main(): particles/s (cold L2 | warm L2) and the
    fraction of the HBM roofline (cold) / of the L2 read bandwidth (warm, L2-resident)."""
    schemes = []
    for r in rows:
        if r["scheme"] not in schemes:
            schemes.append(r["scheme"])
    out = ["# Round 2 sweep: resample-only throughput vs P and weight variance (tools/sweep.py)", "",
           "One B200, `pf_resample_batched` device time per call. **cold**: L2 flushed (512 MiB write) before "
           "every call, inputs from HBM; fraction = library-stated algorithmic bytes / time / "
           f"{hbm:.0f} GB/s (MEASURED_PEAKS hbm_gbs). **warm**: calls replayed back to back in a CUDA graph, so "
           "working sets below L2 stay resident; for those (marked L2) the fraction is of the measured L2 read "
           f"bandwidth {l2 if l2 else float('nan'):.0f} GB/s (`tools/microbench`, `profiles/r02_microbench.md`). "
           "Cells: particles/s cold (frac) / warm (frac). Single filters (N = 1) and batches with N x P = 2^26. "
           "Raw: `profiles/r02_sweep.jsonl`.", ""]
    for batched in (False, True):
        out += ["## " + ("batches (N x P = 2^26)" if batched else "single filter (N = 1)"), "",
                "| P | sigma^2 | " + " | ".join(schemes) + " |", "|---|---|" + "---|" * len(schemes)]
        cells = {}
        for r in rows:
            if r["batched"] == batched:
                cells[(r["P"], r["var"], r["scheme"])] = r
        for P, var in sorted({(k[0], k[1]) for k in cells}):
            lp = P.bit_length() - 1
            vals = []
            for sc in schemes:
                r = cells.get((P, var, sc))
                if not r:
                    vals.append("-")
                    continue
                cf = f" ({r['frac_hbm_cold']:.2f})" if r.get("frac_hbm_cold") is not None else ""
                wf = f" ({r['frac_l2_warm']:.2f} L2)" if r.get("frac_l2_warm") is not None else ""
                vals.append(f"{r['cold_particles_per_s']:.2e}{cf} / {r['warm_particles_per_s']:.2e}{wf}")
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
    hbm, l2 = peaks_from_files()
    scratch = torch.empty(1 << 27, dtype=torch.int32, device=dev)
    rows = []
    cases = [("systematic", 0, 0), ("stratified", 0, 0), ("multinomial", 0, 0),
             ("multinomial", 0, pf.PF_SORTED), ("metropolis", 32, 0)]
    l2_bytes = 60 << 20  # working sets below this stay L2-resident across graph replays
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
                    def fn():
                        pf.pf_resample_batched(scheme, x, 5, B=B, ancestors=anc, flags=flags)
                    reps = 20 if N * P <= (1 << 22) else 5
                    warm = time_calls(fn, reps, dev)
                    cold = cold_time(fn, 10 if N * P <= (1 << 22) else 5, dev, scratch)
                    ab, kern = alg_bytes(pf, fn, dev)
                    name = scheme + ("_sorted_a6" if flags else "") + (f"_B{B}" if B else "")
                    row = {"batched": batched, "N": N, "P": P, "var": var, "scheme": name,
                           "warm_us": round(warm * 1e3, 2), "cold_us": round(cold * 1e3, 2),
                           "warm_particles_per_s": N * P / (warm / 1e3),
                           "cold_particles_per_s": N * P / (cold / 1e3), "alg_bytes": ab, "launches": kern}
                    if ab:
                        row["frac_hbm_cold"] = ab / (cold / 1e3) / 1e9 / hbm
                        if l2 and ab < l2_bytes:
                            row["frac_l2_warm"] = ab / (warm / 1e3) / 1e9 / l2
                    rows.append(row)
                    print(json.dumps(row))
                    sys.stdout.flush()
    if md:
        write_md(rows, md, hbm, l2)


if __name__ == "__main__":
    main()
