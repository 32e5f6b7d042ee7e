#!/usr/bin/env python
"""Throughput sweep over P and weight variance (BASELINE metric "resampled particles/sec
vs P and weight variance"; SURVEY §8(d) companion sweep P = 2^4 ... 2^24).

Single filters (N = 1) and batches with N * P = 2^26 (P <= 2^16), every scheme,
sigma^2 in {0.1, 1, 10}; CUDA events over R back-to-back calls after warm-up
(inputs resident in HBM).  JSON lines on stdout.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


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
                    for _ in range(3):
                        pf.pf_resample_batched(scheme, x, 5, B=B, ancestors=anc, flags=flags, stream=stream)
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    for r in range(reps):
                        pf.pf_resample_batched(scheme, x, 5 + r, B=B, ancestors=anc, flags=flags, stream=stream)
                    e1.record(stream)
                    torch.cuda.synchronize(dev)
                    ms = e0.elapsed_time(e1) / reps
                    name = scheme + ("_sorted_a6" if flags else "") + (f"_B{B}" if B else "")
                    print(json.dumps({"batched": batched, "N": N, "P": P, "var": var, "scheme": name,
                                      "us_per_call": round(ms * 1e3, 2),
                                      "particles_per_s": N * P / (ms / 1e3)}))
                    sys.stdout.flush()


if __name__ == "__main__":
    main()
