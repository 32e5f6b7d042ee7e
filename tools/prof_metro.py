"""Drive the C3 Metropolis resampler (k_mexp + k_metro_fpc, B = 32) for ncu:
  ncu --set full -k regex:k_metro -s 2 -c 1 python tools/prof_metro.py [B]"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1202_6163_b200 as pf
    import pfinputs

    B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    dev = torch.device("cuda:0")
    x = pfinputs.gaussian_logw_torch(1 << 16, 1.0, 3, 1024, dev)
    a = torch.empty((1024, 1 << 16), dtype=torch.int32, device=dev)
    for _ in range(3):
        pf.pf_resample_batched("metropolis", x, 9, B=B, ancestors=a)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
