#!/usr/bin/env python
"""Device time per call (CUDA graph replay) of a few resample configurations; one JSON
line each.  Used to compare build variants (launch geometry) on the same box."""
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
    if "--geom" in sys.argv:
        # systematic batches of N x P = 2^26 by output set (geometry A/B with PF_FUSED_FT)
        for P in (1 << 14, 1 << 15, 1 << 16, 40000):
            N = (1 << 26) // P
            x = pfinputs.gaussian_logw_torch(P, 1.0, pfinputs.BASE_SEED, N, dev)
            anc = torch.empty((N, P), dtype=torch.int32, device=dev)
            off = torch.empty_like(anc)
            pm = torch.empty_like(anc)
            for name, kw in (("anc", {}), ("perm", {"offspring_out": off, "permuted_out": pm})):
                ms = time_calls(lambda: pf.pf_resample_batched("systematic", x, 5, ancestors=anc, **kw), 5, dev)
                print(json.dumps({"P": P, "N": N, "outputs": name, "ms": round(ms, 4),
                                  "particles_per_s": N * P / (ms / 1e3)}))
                sys.stdout.flush()
        return
    if "--c3" in sys.argv:
        # the C3 batch (1024 x 2^16, sigma^2 = 1 unless --var) by output set: resample only,
        # + offspring, + permutation, + in-place gather of a D = 16 state (the bench step)
        var = float(sys.argv[sys.argv.index("--var") + 1]) if "--var" in sys.argv else 1.0
        N, P = 1024, 1 << 16
        x = pfinputs.gaussian_logw_torch(P, var, pfinputs.BASE_SEED, N, dev)
        anc = torch.empty((N, P), dtype=torch.int32, device=dev)
        off = torch.empty_like(anc)
        pm = torch.empty_like(anc)
        X = torch.randn((N, P, 16), device=dev)
        for scheme in ("systematic", "stratified", "multinomial"):
            for name, kw in (("anc", {}), ("off", {"offspring_out": off}),
                             ("perm", {"offspring_out": off, "permuted_out": pm}),
                             ("step", {"offspring_out": off, "permuted_out": pm, "state": X})):
                ms = time_calls(lambda: pf.pf_resample_batched(scheme, x, 5, ancestors=anc, **kw), 5, dev)
                print(json.dumps({"c3": scheme, "var": var, "outputs": name, "ms": round(ms, 4),
                                  "particles_per_s": N * P / (ms / 1e3)}))
                sys.stdout.flush()
        return
    if "--small" in sys.argv:
        for P in (16, 64, 256):
            for scheme in ("systematic", "multinomial", "metropolis"):
                for N in (1, 4, 16, 64, 1024):
                    x = pfinputs.gaussian_logw_torch(P, 1.0, pfinputs.BASE_SEED, N, dev)
                    anc = torch.empty((N, P), dtype=torch.int32, device=dev)
                    b = 32 if scheme == "metropolis" else 0
                    us = round(1e3 * time_calls(lambda: pf.pf_resample_batched(scheme, x, 5, B=b, ancestors=anc), 10,
                                                dev), 2)
                    print(json.dumps({"P": P, "scheme": scheme, "N": N, "us": us}))
                    sys.stdout.flush()
        return
    if "--medium" in sys.argv:
        # k_medium (one CTA per filter) against the cluster kernel (N = 64 vs 65 straddles the
        # k_medium batch limit of stratified/systematic) and against the multi-launch path
        for P in (512, 1024, 2048, 4096, 8192):
            for scheme in ("systematic", "stratified", "multinomial", "metropolis"):
                for N in (1, 16, 64, 1024):
                    x = pfinputs.gaussian_logw_torch(P, 1.0, pfinputs.BASE_SEED, N, dev)
                    anc = torch.empty((N, P), dtype=torch.int32, device=dev)
                    b = 32 if scheme == "metropolis" else 0
                    row = {"P": P, "scheme": scheme, "N": N}
                    for name, fl in (("default", 0), ("unfused", pf.PF_NO_FUSION)):
                        row[name + "_us"] = round(1e3 * time_calls(
                            lambda: pf.pf_resample_batched(scheme, x, 5, B=b, ancestors=anc, flags=fl), 5, dev), 2)
                    print(json.dumps(row))
                    sys.stdout.flush()
        return
    if "--coop-vs-unfused" in sys.argv:
        for P in (1 << 17, 1 << 18, 1 << 20, 1 << 22):
            for N in (1, 2, 4, 8, 16, 64):
                if N * P > (1 << 26):
                    continue
                x = pfinputs.gaussian_logw_torch(P, 1.0, pfinputs.BASE_SEED, N, dev)
                anc = torch.empty((N, P), dtype=torch.int32, device=dev)
                row = {"N": N, "P": P}
                for name, fl in (("default", 0), ("unfused", pf.PF_NO_FUSION)):
                    row[name] = round(time_calls(lambda: pf.pf_resample_batched("systematic", x, 5, ancestors=anc,
                                                                                flags=fl), 5, dev), 4)
                print(json.dumps(row))
                sys.stdout.flush()
        return
    cases = [(1024, 1 << 16, "systematic", True), (1024, 1 << 16, "stratified", True),
             (512, 1 << 17, "systematic", False), (1, 1 << 18, "systematic", False),
             (1, 1 << 20, "systematic", False), (1, 1 << 24, "systematic", False)]
    for N, P, scheme, perm in cases:
        x = pfinputs.gaussian_logw_torch(P, 1.0, pfinputs.BASE_SEED, N, dev)
        anc = torch.empty((N, P), dtype=torch.int32, device=dev)
        off = torch.empty_like(anc)
        pm = torch.empty_like(anc) if perm else None
        ms = time_calls(lambda: pf.pf_resample_batched(scheme, x, 5, ancestors=anc, offspring_out=off,
                                                       permuted_out=pm), 5, dev)
        print(json.dumps({"N": N, "P": P, "scheme": scheme, "perm": perm, "ms": round(ms, 4),
                          "particles_per_s": N * P / (ms / 1e3), "lib": pf._LIB_PATH}))
        sys.stdout.flush()


if __name__ == "__main__":
    main()
