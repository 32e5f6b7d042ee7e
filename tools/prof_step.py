"""Drive the C3 bench step (pf_resample_batched with offspring, permutation and the in-place
D = 16 state gather) for ncu: two warm-up calls, then one:
  ncu --set full -k regex:k_fused_sorted -s 2 -c 1 python tools/prof_step.py [scheme] [var]"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1202_6163_b200 as pf
    import pfinputs

    scheme = sys.argv[1] if len(sys.argv) > 1 else "systematic"
    var = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    dev = torch.device("cuda:0")
    N, P = 1024, 1 << 16
    x = pfinputs.gaussian_logw_torch(P, var, pfinputs.BASE_SEED, N, dev)
    a = torch.empty((N, P), dtype=torch.int32, device=dev)
    off = torch.empty_like(a)
    pm = torch.empty_like(a)
    X = torch.randn((N, P, 16), device=dev)
    for _ in range(3):
        pf.pf_resample_batched(scheme, x, 5, ancestors=a, offspring_out=off, permuted_out=pm, state=X)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
