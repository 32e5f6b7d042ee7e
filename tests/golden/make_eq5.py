"""Writes eq5_required_B.txt with mpmath (50 digits).  Calls nothing under
oracle/ or the product path: it evaluates PAPER.md Eq. (2) and Eq. (5)
 directly, beta = 1/P.  Readings (R-22): B is at least 1
("B = max(1, ceil(Eq. (5)))": a resampler takes at least one step);
w_max < 1/P is outside Eq. (2)'s domain (a maximum of P normalised weights is >= 1/P,
SPEC S:233) and a B beyond int32 cannot be returned: both -> -1."""
import mpmath as mp

mp.mp.dps = 50
CASES = [(1024, "0.1", "0.01"), (1024, "0.1", "0.001"), (2, "1", "0.01"),
         (16, "0.0625", "0.01"), (65536, "0.01", "0.01"), (256, "0.05", "0.01"),
         (4096, "0.002", "0.001"),
         # R-22 edge cases: Eq. (5) already satisfied (bound >= 1) -> 1; w_max < 1/P -> -1;
         # w_max -> 1 at the C5 size: B ~ P ln(1/eps) > 2^31 -> -1; w_max = 1/P exactly (lambda = 0)
         (1024, "0.1", "1"), (1024, "0.0009", "0.01"), (268435456, "0.999999", "0.0001"),
         (268435456, "0.5", "0.01"), (4, "0.25", "0.01")]
lines = ["# P w_max eps -> B  (Eq. (5), P:183-186; alpha Eq. (2) P:163-167; beta=1/P P:161)",
         "# computed by tests/golden/make_eq5.py with mpmath at 50 digits",
         "# note: SPEC.md S:254 quotes B~928 for (1024,0.1,0.01); Eq. (5) gives 459 (DESIGN.md R12)"]
for P, w, e in CASES:
    P = mp.mpf(P); w = mp.mpf(w); e = mp.mpf(e)
    beta = 1 / P
    alpha = (1 - w) / (P * w)
    lam = 1 - alpha - beta
    target = e * (alpha + beta) / max(alpha, beta)
    if w < 1 / P:
        B = -1
    elif lam <= 0 or target >= 1:
        B = 1
    else:
        B = max(1, int(mp.ceil(mp.log(target) / mp.log(lam))))
        if B > 2 ** 31 - 1:
            B = -1
    lines.append(f"{int(P)} {mp.nstr(w, 10)} {mp.nstr(e, 10)} {B}")
open(__file__.replace("make_eq5.py", "eq5_required_B.txt"), "w").write("\n".join(lines) + "\n")
