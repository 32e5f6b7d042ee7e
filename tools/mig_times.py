#!/usr/bin/env python
"""Per-kernel times of the sharded resample + particle migration (C5 shape, one rank):
resample_sharded(assemble=False) + migrate_sharded of D float32 rows, traced with
pf_profile_enable (events around every library launch), plus the step's event time."""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1202_6163_b200 as pf
    import pfinputs
    from paper_1202_6163_b200.shard import SingleComm, migrate_sharded, resample_sharded

    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=1 << 25)
    ap.add_argument("--D", type=int, default=16)
    ap.add_argument("--scheme", default="systematic")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    logw = pfinputs.gaussian_logw_torch(a.P, 1.0, pfinputs.BASE_SEED, 1, dev)[0].contiguous()
    X = torch.randn((a.P, a.D), device=dev)
    comm = SingleComm()

    def step(mig=True):
        anc, info = resample_sharded(a.scheme, logw, a.P, 5, comm=comm, assemble=False)
        if mig:
            migrate_sharded(X, anc, info, comm=comm)

    for mig in (False, True):
        for _ in range(3):
            step(mig)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            step(mig)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"migrate": mig, "ms_per_step": e0.elapsed_time(e1) / a.reps}))
    pf.pf_profile_enable(True)
    pf.pf_profile_collect()
    for _ in range(a.reps):
        step(True)
    torch.cuda.synchronize()
    tr = pf.pf_profile_collect()
    pf.pf_profile_enable(False)
    for k, (n, ms, *_) in sorted(tr.items(), key=lambda kv: -kv[1][1]):
        print(json.dumps({"kernel": k, "launches_per_step": n / a.reps, "ms_per_step": ms / a.reps}))


if __name__ == "__main__":
    main()
