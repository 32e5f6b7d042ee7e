#!/usr/bin/env python
"""e2e step (bench.py e2e: pinned host logw in, permutation out, C3 systematic step) by chunk
count and chaining of HostPipeline; one JSON line each."""
import json, sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_1202_6163_b200 as pf
import pfinputs
from paper_1202_6163_b200.pipeline import HostPipeline
dev = torch.device("cuda:0")
N, P = 1024, 1 << 16
x = pfinputs.gaussian_logw_torch(P, 1.0, pfinputs.BASE_SEED, N, dev)
X = torch.randn((N, P, 16), device=dev)
h = x.cpu().pin_memory()
ho = torch.empty((N, P), dtype=torch.int32).pin_memory()
for chunks in [int(c) for c in (sys.argv[1].split(",") if len(sys.argv) > 1 else "8,16,32,64".split(","))]:
    for chain in (False, True):
        pipe = HostPipeline(N, P, dev, chunks=chunks)
        st = torch.cuda.current_stream(dev)
        for _ in range(2):
            pipe.run("systematic", h, 5, ho, state=X, stream=st, chain=chain)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(10):
            pipe.run("systematic", h, 5, ho, state=X, stream=st, chain=chain)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(json.dumps({"chunks": chunks, "chain": chain, "ms": round(ms, 3), "particles_per_s": N * P / ms * 1e3}))
        del pipe
