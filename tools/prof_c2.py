"""Drive one C2 step (single filter P = 2^20, sigma^2 = 1, systematic, offspring + permutation +
D = 16 state gather; and resample-only) and the C3 sorted multinomial (a6) for ncu:
  ncu --set full -k regex:"k_coop|k_gather|k_gscan|k_merge" python tools/prof_c2.py"""
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
    P = 1 << 20
    x = pfinputs.gaussian_logw_torch(P, 1.0, pfinputs.BASE_SEED, 1, dev)
    anc = torch.empty((1, P), dtype=torch.int32, device=dev)
    off = torch.empty_like(anc)
    pm = torch.empty_like(anc)
    X = torch.randn((1, P, 16), device=dev)
    for _ in range(2):
        pf.pf_resample_batched("systematic", x, 5, ancestors=anc)
        pf.pf_resample_batched("systematic", x, 5, ancestors=anc, offspring_out=off, permuted_out=pm, state=X)
    xb = pfinputs.gaussian_logw_torch(1 << 16, 1.0, pfinputs.BASE_SEED, 1024, dev)
    ab = torch.empty((1024, 1 << 16), dtype=torch.int32, device=dev)
    pf.pf_resample_batched("multinomial", xb, 5, ancestors=ab, flags=pf.PF_SORTED)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
