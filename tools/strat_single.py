#!/usr/bin/env python
"""Stratified single filters of 2^18 / 2^20 / 2^22 / 2^24 (cooperative kernel), ancestors only and
with the permutation: device time per call (graph replay), one JSON line each."""
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
    from tools.sweep import time_calls

    dev = torch.device("cuda:0")
    for lp in (18, 20, 22, 24):
        P = 1 << lp
        x = pfinputs.gaussian_logw_torch(P, 1.0, pfinputs.BASE_SEED, 1, dev)
        anc = torch.empty((1, P), dtype=torch.int32, device=dev)
        off = torch.empty_like(anc)
        pm = torch.empty_like(anc)
        for name, kw in (("anc", {}), ("perm", {"offspring_out": off, "permuted_out": pm})):
            ms = time_calls(lambda: pf.pf_resample_batched("stratified", x, 5, ancestors=anc, **kw), 10, dev)
            print(json.dumps({"P": P, "outputs": name, "ms": round(ms, 4)}))


if __name__ == "__main__":
    main()
