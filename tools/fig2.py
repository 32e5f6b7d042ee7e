#!/usr/bin/env python
"""Fig. 2 of the paper on B200.

Weight sets w ~ Dir(alpha) for P = 256, 512, ..., 65536 and alpha = 10, 1, .1, .01
(pfinputs.dirichlet_logw).  For every (alpha, P) and scheme:

* error: the mean over R resamplings of sum_i (o_i / P - v_i)^2 (the caption of Fig. 2),
  R = 1000 independent resamplings of the same weight set run as ONE batched launch
  (filter index r -> an independent Philox stream), offspring o from pf_opts.offspring_out;
  compared with its closed form: multinomial (1 - sum v^2) / P; systematic
  sum_i f_i (1 - f_i) / P^2 with f_i = frac(P v_i); stratified sum over (particle, stratum)
  overlaps p (1 - p) / P^2; Metropolis -> multinomial's as B grows.
* Metropolis B from Eq. (5) with the set's w_max and eps = .01
  (pf_metropolis_required_B), as the paper tunes it; R is reduced when
  R * P * B would exceed --max-proposals (2e11 by default; reported).
* runtime: device time of ONE resampling call (CUDA graph of repeated calls, as the paper
  times single resamplings) and the amortised time per resampling in the batched launch.

Output: JSON lines on stdout; ``--md FILE`` also writes a markdown summary.
No oracle: closed forms are computed here in float64 from the weights.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SCHEMES = ("multinomial", "sorted_multinomial", "stratified", "systematic", "metropolis")


def closed_forms(v):
    import numpy as np

    P = len(v)
    multi = (1.0 - float(np.sum(v * v))) / P
    f = np.mod(P * v, 1.0)
    syst = float(np.sum(f * (1.0 - f))) / (P * P)
    # stratified: merge particle boundaries c_i with stratum boundaries k / P; each segment
    # of length l belongs to one (particle, stratum) pair with probability p = P l
    c = np.concatenate([[0.0], np.cumsum(v)])
    c[-1] = 1.0
    br = np.unique(np.concatenate([c, np.arange(P + 1) / P]))
    seg = np.diff(br)
    p = np.clip(P * seg, 0.0, 1.0)
    strat = float(np.sum(p * (1.0 - p))) / (P * P)
    return {"multinomial": multi, "sorted_multinomial": multi, "metropolis": multi, "stratified": strat,
            "systematic": syst}


def main():
    import numpy as np
    import torch

    import paper_1202_6163_b200 as pf
    import pfinputs
    from tools.sweep import time_calls

    ap = argparse.ArgumentParser()
    ap.add_argument("--R", type=int, default=1000)
    ap.add_argument("--eps", type=float, default=0.01)
    ap.add_argument("--max-proposals", type=float, default=2e11)
    ap.add_argument("--md", default=None)
    ap.add_argument("--quick", action="store_true", help="P <= 4096 only")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    rows = []
    Ps = [256 << k for k in range(9)]
    if a.quick:
        Ps = [p for p in Ps if p <= 4096]
    for alpha in (10.0, 1.0, 0.1, 0.01):
        for P in Ps:
            x = pfinputs.dirichlet_logw(P, alpha, seed=int(1000 * alpha) + P)
            xd = x.astype(np.float64)
            v = np.exp(xd - xd.max())
            v /= v.sum()
            ess = 1.0 / float(np.sum(v * v))
            cf = closed_forms(v)
            B = max(0, pf.pf_metropolis_required_B(P, float(v.max()), a.eps))
            g1 = torch.from_numpy(x).to(dev)
            for scheme in SCHEMES:
                name = "multinomial" if scheme == "sorted_multinomial" else scheme
                flags = pf.PF_SORTED if scheme == "sorted_multinomial" else 0
                b = B if scheme == "metropolis" else 0
                R = a.R
                if scheme == "metropolis":
                    R = int(max(8, min(a.R, a.max_proposals / max(1.0, float(P) * max(b, 1)))))
                G = g1.expand(R, P)  # the same weight set R times
                G = G.contiguous()
                off = torch.empty((R, P), dtype=torch.int32, device=dev)
                t_batch = time_calls(lambda: pf.pf_resample_batched(name, G, 11, B=b, offspring_out=off,
                                                                    flags=flags), 1, dev)
                pf.pf_resample_batched(name, G, 11, B=b, offspring_out=off, flags=flags)
                torch.cuda.synchronize()
                o = off.to(torch.float64) / P
                vt = torch.from_numpy(v).to(dev)
                err = ((o - vt) ** 2).sum(dim=1)
                e_mean = float(err.mean())
                e_sem = float(err.std() / math.sqrt(R)) if R > 1 else float("nan")
                anc1 = torch.empty(P, dtype=torch.int32, device=dev)
                reps = 20 if P * max(b, 1) <= (1 << 24) else 3
                t_one = time_calls(lambda: pf.pf_resample_ex(name, g1, 7, b, ancestors=anc1, flags=flags), reps, dev)
                row = {"alpha": alpha, "P": P, "scheme": scheme, "B": b, "R": R, "ess_over_P": ess / P,
                       "error_mean": e_mean, "error_sem": e_sem, "error_closed_form": cf[scheme],
                       "us_per_resampling_single": round(1e3 * t_one, 3),
                       "us_per_resampling_batched": round(1e3 * t_batch / R, 4)}
                rows.append(row)
                print(json.dumps(row))
                sys.stdout.flush()
    if a.md:
        write_md(rows, a)


def write_md(rows, a):
    by = {}
    for r in rows:
        by.setdefault((r["alpha"], r["P"]), {})[r["scheme"]] = r
    out = ["# Fig. 2 on B200 (P:191-250; `tools/fig2.py`)", "",
           f"Dirichlet weights, 1000 resamplings per cell (Metropolis: fewer where R P B > "
           f"{a.max_proposals:.0e} proposals, column R), Metropolis B from Eq. (5) with eps = {a.eps}. "
           "Error = mean over resamplings of sum_i (o_i/P - v_i)^2 (x 1e-6), measured / closed form. "
           "Time = device time of one resampling call (us) | amortised per resampling in the batched launch (us).",
           ""]
    for alpha in sorted({k[0] for k in by}, reverse=True):
        out += [f"## alpha = {alpha:g}", "",
                "| P | ESS/P | multinomial err | stratified err | systematic err | Metropolis err (B, R) | "
                "time: multinomial | sorted multi. | stratified | systematic | Metropolis |",
                "|---|---|---|---|---|---|---|---|---|---|---|"]
        for P in sorted(p for (al, p) in by if al == alpha):
            c = by[(alpha, P)]

            def e(s):
                return f"{1e6 * c[s]['error_mean']:.3g} / {1e6 * c[s]['error_closed_form']:.3g}"

            def t(s):
                return f"{c[s]['us_per_resampling_single']:.1f} \\| {c[s]['us_per_resampling_batched']:.3f}"

            m = c["metropolis"]
            out.append(f"| {P} | {c['systematic']['ess_over_P']:.3f} | {e('multinomial')} | {e('stratified')} | "
                       f"{e('systematic')} | {e('metropolis')} ({m['B']}, {m['R']}) | {t('multinomial')} | "
                       f"{t('sorted_multinomial')} | {t('stratified')} | {t('systematic')} | {t('metropolis')} |")
        out.append("")
    with open(a.md, "w") as f:
        f.write("\n".join(out) + "\n")


if __name__ == "__main__":
    main()
