"""Drive the resample-only cluster kernel (k_fused_sorted<SCHEME, 0, 0>) at C3 (1024 x 2^16)
for ncu: two warm-up calls, then one:
  ncu --set full -k regex:k_fused_sorted -s 2 -c 1 python tools/prof_resample_only.py [scheme]"""
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
    dev = torch.device("cuda:0")
    x = pfinputs.gaussian_logw_torch(1 << 16, 1.0, 1, 1024, dev)
    a = torch.empty_like(x, dtype=torch.int32)
    for _ in range(3):
        pf.pf_resample_batched(scheme, x, 3, ancestors=a)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
