#!/usr/bin/env python
"""Per-kernel device times of the C4 bootstrap-PF step (pf_profile_enable, CUDA events on the
launching stream): where the ~55 us per step go."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1202_6163_b200 as pf
    import pfinputs
    from paper_1202_6163_b200.pf_demo import LinearGaussianPF

    P = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
    ys = pfinputs.lg_observations(60)
    f = LinearGaussianPF(P, scheme="systematic")
    for y in ys[:10]:
        f.step(float(y))
    torch.cuda.synchronize()
    pf.pf_profile_enable(True)
    for y in ys[10:60]:
        f.step(float(y))
    kt = pf.pf_profile_collect()
    pf.pf_profile_enable(False)
    torch.cuda.synchronize()
    out = {k: {"launches_per_step": c / 50, "us_per_step": 1e3 * t / 50} for k, (c, t, *_) in kt.items()}
    print(json.dumps({"P": P, "kernels": out, "sum_us": sum(v["us_per_step"] for v in out.values())}))


if __name__ == "__main__":
    main()
