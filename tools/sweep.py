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


def main():
    import torch

    import paper_1202_6163_b200 as pf
    import pfinputs

    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
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
                    print(json.dumps({"batched": batched, "N": N, "P": P, "var": var, "scheme": name,
                                      "us_per_call": round(ms * 1e3, 2),
                                      "particles_per_s": N * P / (ms / 1e3)}))
                    sys.stdout.flush()


if __name__ == "__main__":
    main()
