"""Drive the binary64 pre-pass (k_max64 / k_shift64) and the pre-sorted weight sort (k_rhist /
k_rscan / k_rscatter) once at the C3 size (1024 filters x 2^16) after a warm-up, for ncu:
  ncu --set full -k regex:'k_max64|k_shift64|k_rhist|k_rscan|k_rscatter' -s 12 -c 6 python tools/prof_new.py
"""
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
    N, P = 1024, 1 << 16
    x = pfinputs.gaussian_logw_torch(P, 1.0, 1, N, dev)
    x64 = x.double() - 1e7
    a = torch.empty((N, P), dtype=torch.int32, device=dev)
    for _ in range(2):
        pf.pf_resample_batched("systematic", x64, 3, ancestors=a)
        pf.pf_resample_batched("systematic", x, 3, ancestors=a, flags=pf.PF_SORT_WEIGHTS)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
