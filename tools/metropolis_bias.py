#!/usr/bin/env python
"""Metropolis bias report at each B (BASELINE north star "the bias of the
Metropolis resampler reported at each B").

For P = 2^20 single filters with Gaussian log-weights (sigma^2 in {0.1, 1, 10}) and
B in {8, 32, 128} (plus the Eq. (5) B at eps = .01 when it is <= 4096), R replicates
over seeds on the GPU (libpfresample), reported per (sigma^2, B):
  * mean offspring of the max particle / P  vs  the corrected Eq. (3) closed form
    (R-11)  vs  w_max (the converged value)
  * mean Fig. 2 error sum_i (o_i/P - v_i)^2 vs the multinomial's (1 - sum v^2)/P
  * the systematic, stratified and multinomial errors on the same inputs
Writes JSON lines to stdout.
"""
from __future__ import annotations

import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1202_6163_b200 as pf
    import pfinputs

    dev = torch.device("cuda:0")
    P = int(os.environ.get("PF_BIAS_P", 1 << 20))
    R = int(os.environ.get("PF_BIAS_R", 64))
    for var in (0.1, 1.0, 10.0):
        x = pfinputs.gaussian_logw_torch(P, var, pfinputs.BASE_SEED, 1, dev)[0].contiguous()
        v = torch.softmax(x.double(), 0)
        imax = int(torch.argmax(v).item())
        wmax = float(v[imax].item())
        sum_v2 = float((v * v).sum().item())
        alpha = (1.0 - wmax) / (P * wmax)  # Eq. (2)
        beta = 1.0 / P
        lam = 1.0 - alpha - beta
        Beq5 = pf.pf_metropolis_required_B(P, wmax, 0.01)
        errs = {}
        for scheme in ("multinomial", "stratified", "systematic"):
            e = []
            for r in range(R):
                a = pf.pf_resample_ex(scheme, x, pfinputs.seed_for(r))
                o = torch.bincount(a.long(), minlength=P).double()
                e.append(float(((o / P - v) ** 2).sum().item()))
            errs[scheme] = sum(e) / R
        Bs = [8, 32, 128] + ([Beq5] if 0 < Beq5 <= 4096 else [])
        for B in Bs:
            omax, e = [], []
            for r in range(R):
                a = pf.pf_resample_metropolis(x, pfinputs.seed_for(1000 + r), B)
                o = torch.bincount(a.long(), minlength=P).double()
                omax.append(float(o[imax].item()))
                e.append(float(((o / P - v) ** 2).sum().item()))
            s = alpha + beta
            closed = (beta / s + lam ** B * alpha / s) + (P - 1) * (beta / s) * (1 - lam ** B)
            mean_omax = sum(omax) / R
            sd = math.sqrt(sum((t - mean_omax) ** 2 for t in omax) / max(R - 1, 1))
            print(json.dumps({
                "P": P, "var": var, "B": B, "replicates": R, "w_max": wmax, "ess_over_P": 1.0 / sum_v2 / P,
                "eq5_B_eps0.01": Beq5,
                "omax_over_P_measured": mean_omax / P, "omax_over_P_se": sd / math.sqrt(R) / P,
                "omax_over_P_closed_form_eq3": closed / P, "converged_value_w_max": wmax,
                "bias_of_omax_vs_w_max": mean_omax / P - wmax,
                "fig2_error_metropolis": sum(e) / R,
                "fig2_error_multinomial_closed_form": (1 - sum_v2) / P,
                "fig2_error_measured": errs,
            }))
            sys.stdout.flush()


if __name__ == "__main__":
    main()
