#!/usr/bin/env python
"""Drive the cooperative kernel on one 2^24 filter with offspring + permutation (the p24 step's
resampling launch) for ncu: two warm-up calls, then one:
  ncu --set full -k regex:k_coop -s 2 -c 1 python tools/prof_p24.py"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1202_6163_b200 as pf
    import pfinputs

    dev = torch.device("cuda:0")
    x = pfinputs.gaussian_logw_torch(1 << 24, 1.0, 1, 1, dev)
    a = torch.empty_like(x, dtype=torch.int32)
    o = torch.empty_like(a)
    p = torch.empty_like(a)
    for _ in range(3):
        pf.pf_resample_batched("systematic", x, 3, ancestors=a, offspring_out=o, permuted_out=p)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
