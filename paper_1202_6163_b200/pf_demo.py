"""Bootstrap particle filter on the linear-Gaussian demo model (BASELINE config C4;
PAPER.md P:43-68: initialise, propagate, weight, resample).

Every step runs in libpfresample kernels: pf_lg_propagate_weight (steps 2-3),
pf_resample_ex (step 4: lse + offspring side outputs), pf_lg_accumulate (log
of the likelihood increment), pf_permute_offspring + pf_gather_state (the
resampled population in place).  Host code only sequences the calls.
"""
from __future__ import annotations

_M64 = (1 << 64) - 1


def step_seed(seed: int, t: int) -> int:
    """splitmix64(seed + t): a fresh resampling key per time step."""
    x = (seed + t + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


class LinearGaussianPF:
    def __init__(self, P: int, D: int = 16, phi: float = 0.9, sigma_x: float = 1.0, sigma_y: float = 1.0,
                 scheme: str = "systematic", B: int = 0, seed: int = 1, device="cuda:0"):
        import torch

        import paper_1202_6163_b200 as pf

        self.pf, self.torch = pf, torch
        self.P, self.D, self.phi, self.sx, self.sy = P, D, phi, sigma_x, sigma_y
        self.scheme, self.B, self.seed = scheme, B, seed
        dev = torch.device(device)
        self.X = torch.empty((P, D), dtype=torch.float32, device=dev)
        self.logw = torch.empty(P, dtype=torch.float32, device=dev)
        self.anc = torch.empty(P, dtype=torch.int32, device=dev)
        self.off = torch.empty(P, dtype=torch.int32, device=dev)
        self.perm = torch.empty(P, dtype=torch.int32, device=dev)
        self.lse = torch.zeros(1, dtype=torch.float64, device=dev)
        self.loglik = torch.zeros(1, dtype=torch.float64, device=dev)
        self.t = 0
        pf.pf_lg_init(self.X, phi, sigma_x, seed)

    def step(self, y: float, check: bool = False):
        """One filter step; with check=True returns (logw, ancestors, resampling seed) of this step
        (host copies, for the parity test)."""
        pf = self.pf
        self.t += 1
        pf.pf_lg_propagate_weight(self.X, self.phi, self.sx, self.sy, y, self.seed, self.t, self.logw)
        logw_snap = self.logw.cpu().numpy() if check else None
        # resample (lse, offspring, canonical permutation) and gather the state in place: one launch
        # of the cluster kernel for stratified / systematic up to P = 2^18
        pf.pf_resample_ex(self.scheme, self.logw, step_seed(self.seed, self.t), self.B, ancestors=self.anc,
                          lse_out=self.lse, offspring_out=self.off, permuted_out=self.perm, state=self.X)
        snap = (logw_snap, self.anc.cpu().numpy(), step_seed(self.seed, self.t)) if check else None
        pf.pf_lg_accumulate(self.lse, self.P, self.sy, self.loglik)
        return snap

    def run(self, ys):
        for y in ys:
            self.step(float(y))
        return float(self.loglik.item())
