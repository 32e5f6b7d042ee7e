"""Element-wise oracle of the C4 demo model's propagate / weight step (TEST INFRASTRUCTURE;
imported only by tests/, __graft_entry__.smoke() and bench.py's reference arm).

DESIGN.md R-20 / NS-18: diagonal AR(1) in D dimensions, x_t = phi x_{t-1} + sigma_x eps_t,
y_t = x_t[0] + sigma_y eta_t (the bootstrap filter's proposal is the transition, so the
incremental log-weight is the observation log-density up to a constant):
    logw_i = -(y_t - x_t,i[0])^2 / (2 sigma_y^2).
The noise of particle i, time t, dimensions 4b..4b+3 comes from (r0..r3) = Philox4x32-10
(c0 = i, c1 = t * ceil(D/4) + b, tag 6, filter 0) (initial state: c1 = b, tag 7, scale
sigma_x / sqrt(1 - phi^2)); uniforms u_q = fl32(fl32(r_q) + 1/2) 2^-32 (binary32, as the design
fixes them); Box-Muller in real arithmetic (here binary64):
    z = (sqrt(-2 ln u0) cos 2 pi u1, sqrt(-2 ln u0) sin 2 pi u1,
         sqrt(-2 ln u2) cos 2 pi u3, sqrt(-2 ln u2) sin 2 pi u3).
The GPU evaluates the same expressions in binary32 with library functions of <= 2 ulp, so the
comparison is element-wise within a tolerance (tests/test_gpu_parity.py), not bit-exact.
Pinned (tests/test_oracle_pins.py) by the standard-normal law of z and the AR(1) moments."""
from __future__ import annotations

import math

import numpy as np

from . import philox


def _key(seed: int):
    return [seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF]


def _uniforms(r) -> np.ndarray:
    r32 = np.asarray(r, dtype=np.uint32).astype(np.float32)
    return ((r32 + np.float32(0.5)) * np.float32(2.0 ** -32)).astype(np.float64)


def box_muller4(r) -> np.ndarray:
    u = _uniforms(r)
    a = math.sqrt(-2.0 * math.log(u[0]))
    b = math.sqrt(-2.0 * math.log(u[2]))
    return np.array([a * math.cos(2 * math.pi * u[1]), a * math.sin(2 * math.pi * u[1]),
                     b * math.cos(2 * math.pi * u[3]), b * math.sin(2 * math.pi * u[3])])


def noise(i: int, c1: int, tag: int, seed: int) -> np.ndarray:
    return box_muller4(philox([i, c1, tag, 0], _key(seed)))


def lg_init(P: int, D: int, phi: float, sigma_x: float, seed: int) -> np.ndarray:
    """x_0 ~ stationary N(0, sigma_x^2 / (1 - phi^2)) per dimension (R-20), binary64."""
    sd = sigma_x / math.sqrt(1.0 - phi * phi)
    nb = -(-D // 4)
    X = np.zeros((P, D))
    for i in range(P):
        z = np.concatenate([noise(i, b, 7, seed) for b in range(nb)])
        X[i] = sd * z[:D]
    return X


def lg_step(X: np.ndarray, y: float, t: int, phi: float, sigma_x: float, sigma_y: float, seed: int):
    """One propagate + weight step from state X [P, D]: returns (X_t, logw) in binary64."""
    P, D = X.shape
    nb = -(-D // 4)
    Xn = np.empty((P, D))
    for i in range(P):
        z = np.concatenate([noise(i, t * nb + b, 6, seed) for b in range(nb)])
        Xn[i] = phi * X[i].astype(np.float64) + sigma_x * z[:D]
    logw = -((y - Xn[:, 0]) ** 2) / (2.0 * sigma_y * sigma_y)
    return Xn, logw
