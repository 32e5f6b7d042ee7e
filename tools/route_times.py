#!/usr/bin/env python
"""Per-rank work of the giant filter's unsorted multinomial (C5): the
replicated search (pf_shard_search: every rank generates all P_global positions) against the
routed stages (pf_shard_route_count + pack for the rank's own slot shard, + search of the
positions routed to it), for rank 0 of G fake shards of 2^25 particles each on one GPU (the
exchanges by slicing, outside the timed region).  One JSON line per G."""
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
    from paper_1202_6163_b200.shard import GpuStages, shard_range

    dev = torch.device("cuda:0")
    st = GpuStages()
    per = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 25
    seed, fi = 77, 0
    for G in (1, 2, 4, 8):
        P = per * G
        x = pfinputs.gaussian_logw_torch(P, 1.0, pfinputs.BASE_SEED, 1, dev)[0].contiguous()
        parts = [shard_range(P, G, g) for g in range(G)]
        mx = [st.max(x[p0:p0 + Pl]) for p0, Pl in parts]
        gmax = torch.stack([m for m, _ in mx]).max(dim=0).values
        gbad = torch.stack([b for _, b in mx]).max(dim=0).values
        scans = [st.scan(x[p0:p0 + Pl], P, gmax) for p0, Pl in parts]
        totals = torch.cat([t for _, t, _ in scans])
        Q0 = scans[0][0]
        anc = torch.full((P,), -1, dtype=torch.int32, device=dev)
        # what rank 0 receives (prepared untimed)
        cnts = [st.route_count(totals, g, P, gmax, gbad, seed, fi) for g in range(G)]
        M = torch.stack(cnts).cpu().tolist()
        packs = [st.route_pack(totals, g, P, gmax, gbad, seed, fi, cnts[g], sum(M[g])) for g in range(G)]
        rx = torch.cat([packs[g][0][0:M[g][0]] for g in range(G)])
        rk = torch.cat([packs[g][1][0:M[g][0]] for g in range(G)])

        def timed(fn, reps=5):
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / reps

        rep_ms = timed(lambda: st.search(1, Q0, 0, P, totals, 0, gmax, gbad, seed, fi, anc))
        cnt_ms = timed(lambda: st.route_count(totals, 0, P, gmax, gbad, seed, fi))
        pack_ms = timed(lambda: st.route_pack(totals, 0, P, gmax, gbad, seed, fi, cnts[0], sum(M[0])))
        srch_ms = timed(lambda: st.route_search(Q0, 0, P, totals, 0, gmax, gbad, rx, rk, anc))
        print(json.dumps({"G": G, "P_global": P, "rank0_particles": parts[0][1], "replicated_search_ms": round(rep_ms, 4),
                          "routed_count_ms": round(cnt_ms, 4), "routed_pack_ms": round(pack_ms, 4),
                          "routed_search_ms": round(srch_ms, 4),
                          "routed_total_ms": round(cnt_ms + pack_ms + srch_ms, 4), "received": int(rx.shape[0])}))
        sys.stdout.flush()
        del x, scans, anc, packs, rx, rk
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
