"""Exact filter for the C4 demo model (TEST INFRASTRUCTURE).

DESIGN.md R-20: diagonal AR(1) state x_t = phi x_{t-1} + sigma_x eps_t in D
dimensions, stationary start, observation y_t = x_t[0] + sigma_y eta_t.  Only
dimension 0 is observed, so the marginal likelihood p(y_1:T) is that of the
scalar Kalman filter on dimension 0 (textbook recursion, plain numpy)."""
from __future__ import annotations

import math


def kalman_loglik(ys, phi=0.9, sigma_x=1.0, sigma_y=1.0):
    m, v = 0.0, sigma_x ** 2 / (1.0 - phi ** 2)  # x_0 stationary
    ll = 0.0
    means = []
    for y in ys:
        mp, vp = phi * m, phi * phi * v + sigma_x ** 2  # predict
        S = vp + sigma_y ** 2
        ll += -0.5 * (math.log(2 * math.pi * S) + (y - mp) ** 2 / S)
        K = vp / S
        m, v = mp + K * (y - mp), (1 - K) * vp
        means.append(m)
    return ll, means
