"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py.  Holds NONE of the method's arithmetic (no exp, no scan, no search):
it only draws log-weights / states and derives per-replicate seeds.

Recipe:
  * Gaussian log-weights logw_i = sigma * z_i, z ~ N(0,1) from numpy PCG64,
    cast to float32; sigma^2 in {0.1, 1, 10}.
  * Paper-matched Dirichlet(alpha) weights as log Gamma(alpha)
    draws: logw_i = log G_i, G_i ~ Gamma(alpha), drawn in log space (no underflow
    at alpha = .01); normalisation is irrelevant to every scheme: only ratios
    enter.
  * Edge-case sets: all-equal, single support (-inf elsewhere), runs of -inf,
    NaN / +inf / all -inf (invalid).
  * Replicate r uses resampling seed splitmix64(BASE_SEED + r).
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 0x12026163
_M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """Vigna's splitmix64 finaliser (seed derivation only)."""
    x = (x + 0x9E3779B97F4A7C15) & _M64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def seed_for(replicate: int, base: int = BASE_SEED) -> int:
    return splitmix64(base + replicate)


def gaussian_logw(P: int, var: float = 1.0, seed: int = BASE_SEED, N: int | None = None) -> np.ndarray:
    """float32 logw of shape (P,) or (N, P): sqrt(var) * N(0,1)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    shape = (P,) if N is None else (N, P)
    z = rng.standard_normal(size=shape, dtype=np.float32)
    return (np.float32(np.sqrt(var)) * z).astype(np.float32)


def gaussian_logw_torch(P: int, var: float, seed: int, N: int, device):
    """Same distribution generated directly on a torch device (bench-size inputs;
    parity at bench size is checked on sampled outputs against numpy copies)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    z = torch.randn((N, P), generator=g, device=device, dtype=torch.float32)
    return z * float(np.sqrt(var))


def dirichlet_logw(P: int, alpha: float, seed: int = BASE_SEED) -> np.ndarray:
    """log G_i, G_i ~ Gamma(alpha), drawn in log space so that small alpha does not
    underflow to zero weights: G_alpha = G_{alpha+1} U^{1/alpha} (Marsaglia & Tsang),
    so log G = log G_{alpha+1} + log(U) / alpha (same law)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    g1 = rng.standard_gamma(alpha + 1.0, size=P)
    u = rng.random(size=P)
    with np.errstate(divide="ignore"):
        return (np.log(g1) + np.log(u) / alpha).astype(np.float32)


def equal_logw(P: int, value: float = 0.0) -> np.ndarray:
    return np.full(P, value, dtype=np.float32)


def single_support_logw(P: int, index: int) -> np.ndarray:
    x = np.full(P, -np.inf, dtype=np.float32)
    x[index] = 0.0
    return x


def with_neg_inf_runs(logw: np.ndarray, frac: float = 0.3, seed: int = 7) -> np.ndarray:
    """Replace random runs of entries by -inf (zero weight), keeping >= 1 finite."""
    rng = np.random.Generator(np.random.PCG64(seed))
    x = logw.copy()
    P = x.shape[-1]
    n_runs = max(1, int(P * frac / 16))
    for _ in range(n_runs):
        s = int(rng.integers(0, P))
        x[..., s:s + int(rng.integers(1, 32))] = -np.inf
    flat = x.reshape(-1, P)
    for row in flat:
        if not np.isfinite(row).any():
            row[0] = 0.0
    return x


def state_matrix(P: int, D: int, seed: int = BASE_SEED) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed ^ 0x5A5A))
    return rng.standard_normal(size=(P, D), dtype=np.float32)


def lg_observations(T: int, phi: float = 0.9, sigma_x: float = 1.0, sigma_y: float = 1.0, D: int = 16,
                    seed: int = BASE_SEED) -> np.ndarray:
    """Observation sequence y_1..y_T simulated from the C4 model (R-20)."""
    rng = np.random.Generator(np.random.PCG64(seed ^ 0xC4))
    x = rng.standard_normal(D) * sigma_x / np.sqrt(1 - phi * phi)
    ys = np.zeros(T)
    for t in range(T):
        x = phi * x + sigma_x * rng.standard_normal(D)
        ys[t] = x[0] + sigma_y * rng.standard_normal()
    return ys


def gaussian_logw_f64(P: int, var: float = 1.0, offset: float = 0.0, seed: int = BASE_SEED,
                      N: int | None = None) -> np.ndarray:
    """binary64 logw = offset + sqrt(var) * z, z ~ N(0,1) in float64: log-weights that carry a
    large common offset (e.g. an accumulated log-likelihood, offset ~ -1e7), the case the
    double-precision entry points (NS-3d, R-21) exist for."""
    rng = np.random.Generator(np.random.PCG64(seed))
    shape = (P,) if N is None else (N, P)
    return offset + np.sqrt(var) * rng.standard_normal(size=shape)


def grid_logw(P: int, var: float = 1.0, seed: int = BASE_SEED, N: int | None = None) -> np.ndarray:
    """float32 Gaussian log-weights rounded to multiples of 2^-12 (|x| < 2^11): adding a
    power-of-two offset up to 2^40 to them is exact in binary64 and their differences are
    exact in binary32 (the exact-shift pins of NS-3d)."""
    x = gaussian_logw(P, var, seed, N).astype(np.float64)
    return (np.clip(np.round(x * 4096.0), -(2 ** 22) + 1, 2 ** 22 - 1) / 4096.0).astype(np.float32)
