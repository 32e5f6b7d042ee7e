"""Writes eq5_required_B.txt with mpmath (50 digits).  Calls nothing under
oracle/ or the product path: it evaluates PAPER.md Eq. (2) and Eq. (5)
 directly, beta = 1/P."""
import mpmath as mp

mp.mp.dps = 50
CASES = [(1024, "0.1", "0.01"), (1024, "0.1", "0.001"), (2, "1", "0.01"),
         (16, "0.0625", "0.01"), (65536, "0.01", "0.01"), (256, "0.05", "0.01"),
         (4096, "0.002", "0.001")]
lines = ["# P w_max eps -> B  (Eq. (5), P:183-186; alpha Eq. (2) P:163-167; beta=1/P P:161)",
         "# computed by tests/golden/make_eq5.py with mpmath at 50 digits",
         "# note: SPEC.md S:254 quotes B~928 for (1024,0.1,0.01); Eq. (5) gives 459 (DESIGN.md R12)"]
for P, w, e in CASES:
    P = mp.mpf(P); w = mp.mpf(w); e = mp.mpf(e)
    beta = 1 / P
    alpha = (1 - w) / (P * w)
    lam = 1 - alpha - beta
    target = e * (alpha + beta) / max(alpha, beta)
    if lam == 0:
        B = 1
    else:
        B = int(mp.ceil(mp.log(target) / mp.log(lam)))
    lines.append(f"{int(P)} {mp.nstr(w, 10)} {mp.nstr(e, 10)} {B}")
open(__file__.replace("make_eq5.py", "eq5_required_B.txt"), "w").write("\n".join(lines) + "\n")
