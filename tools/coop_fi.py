"""A/B of the cooperative kernel's particles per thread (PF_COOP_FI): device time per call
(CUDA graph) of single large filters, resample only and with lse + offspring + permutation.
  PF_COOP_FI=8 python tools/coop_fi.py; PF_COOP_FI=16 python tools/coop_fi.py"""
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
    out = {"PF_COOP_FI": os.environ.get("PF_COOP_FI", "auto")}
    for lg in (17, 18, 19, 20, 21, 22, 24):
        P = 1 << lg
        x = pfinputs.gaussian_logw_torch(P, 1.0, 5, 1, dev)[0].contiguous()
        a = torch.empty(P, dtype=torch.int32, device=dev)
        off = torch.empty(P, dtype=torch.int32, device=dev)
        perm = torch.empty(P, dtype=torch.int32, device=dev)
        lse = torch.empty(1, dtype=torch.float64, device=dev)
        t0 = time_calls(lambda: pf.pf_resample_ex("systematic", x, 3, ancestors=a), 20, dev)
        t1 = time_calls(lambda: pf.pf_resample_ex("systematic", x, 3, ancestors=a, lse_out=lse, offspring_out=off,
                                                  permuted_out=perm), 20, dev)
        t2 = time_calls(lambda: pf.pf_resample_ex("stratified", x, 3, ancestors=a), 20, dev)
        out[f"2^{lg}"] = {"sys_us": round(1e3 * t0, 2), "sys_perm_us": round(1e3 * t1, 2), "strat_us": round(1e3 * t2, 2)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
