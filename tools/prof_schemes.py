"""Run each scheme's batched resample on the C3 workload (for ncu captures)."""
import sys
import torch
import paper_1202_6163_b200 as pf
import pfinputs
dev = torch.device("cuda:0")
N, P = 1024, 1 << 16
x = pfinputs.gaussian_logw_torch(P, 1.0, pfinputs.BASE_SEED, N, dev)
anc = torch.empty((N, P), dtype=torch.int32, device=dev)
for sch in sys.argv[1:] or ["multinomial", "metropolis"]:
    for _ in range(2):
        pf.pf_resample_batched(sch, x, 7, B=32 if sch == "metropolis" else 0, ancestors=anc)
torch.cuda.synchronize()
print("ok")
