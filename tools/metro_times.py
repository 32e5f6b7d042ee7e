#!/usr/bin/env python
"""Device time per batched Metropolis call (CUDA graph) for a few (N, P, B)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_1202_6163_b200 as pf
    import pfinputs
    from tools.sweep import time_calls
    dev = torch.device("cuda:0")
    for N, P, B in ((1024, 1 << 16, 32), (1024, 1 << 16, 8), (1024, 1 << 16, 128), (1024, 1 << 15, 32), (2048, 1 << 14, 32), (148, 1 << 17, 32), (1, 1 << 20, 8), (1, 1 << 20, 32), (1, 1 << 20, 128)):
        x = pfinputs.gaussian_logw_torch(P, 1.0, 3, N, dev)
        anc = torch.empty((N, P), dtype=torch.int32, device=dev)
        ms = time_calls(lambda: pf.pf_resample_batched("metropolis", x, 9, B=B, ancestors=anc), 3, dev)
        print(json.dumps({"N": N, "P": P, "B": B, "ms": round(ms, 4), "proposals_per_s": N * P * B / (ms / 1e3)}))


if __name__ == "__main__":
    main()
