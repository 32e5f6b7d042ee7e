"""Pins of the CPU oracle against what the paper, public known-answer vectors and
mathematics fix — never against the oracle itself.

Each test names the passage (P:n = PAPER.md line n, S:n = SPEC.md line n,
NS-n / R-n = DESIGN.md numeric spec / readings) and the mistake it would catch.
"""
from __future__ import annotations

import math
import os
from fractions import Fraction

import numpy as np
import pytest

import pfinputs
from tests import _philox_py as phx

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


def _lines(path):
    with open(path) as f:
        return [l.strip() for l in f if l.strip() and not l.startswith("#")]


# --------------------------------------------------------------------------- NS-6
def test_philox_kat(orc, golden_dir):
    """NS-6: Random123 known-answer vectors (catches a wrong round, constant or key schedule)."""
    for line in _lines(os.path.join(golden_dir, "philox4x32_10_kat.txt")):
        v = [int(x, 16) for x in line.split()]
        ctr, key, want = v[0:4], v[4:6], v[6:10]
        assert list(orc.philox(ctr, key)) == want
        assert phx.philox4x32_10(ctr, key) == want  # the brute-force helper is pinned too


# --------------------------------------------------------------------------- NS-4
def test_dexp_accuracy_and_special_values(orc):
    """NS-4: <= 2 ulp of exp (math.exp in double) over [-88, 0]; dexp(0)=1; -inf -> 0;
    explicit flush below 2^-126; never above 1 (catches a wrong coefficient or reduction)."""
    rng = np.random.default_rng(1)
    t = np.concatenate([
        -rng.uniform(0, 88, 60000), -rng.uniform(0, 1, 20000), -rng.uniform(0, 1e-6, 5000),
        -np.arange(0, 88, 0.5 * math.log(2)),  # reduction boundaries n*ln2/2
    ]).astype(np.float32)
    d = orc.dexp_array(t)
    e = np.exp(t.astype(np.float64))
    normal = e >= 2.0 ** -126
    ulp = np.spacing(e.astype(np.float32)).astype(np.float64)
    err = np.abs(d.astype(np.float64) - e) / ulp
    assert err[normal].max() <= 2.0, err[normal].max()
    assert np.all((d[~normal] == 0) | (d[~normal] >= 2.0 ** -126))
    assert np.all(d <= 1.0)
    assert orc.dexp(0.0) == 1.0 and orc.dexp(-0.0) == 1.0
    assert orc.dexp(float("-inf")) == 0.0
    assert orc.dexp(-1e-40) == 1.0  # subnormal t
    assert orc.dexp(-88.5) == 0.0 and orc.dexp(-87.2) > 0.0
    # monotone nondecreasing in t on a dense grid
    g = np.sort(-rng.uniform(0, 30, 20000).astype(np.float32))
    dg = orc.dexp_array(g)
    assert np.all(np.diff(dg.astype(np.float64)) >= 0)


# --------------------------------------------------------------------------- NS-1..5
def test_quantise_and_scan_against_exp(orc):
    """NS-5: Q_i - Q_{i-1} = trunc(w_i 2^kfx) with w_i ~ exp(logw_i - lmax); the max particle
    has q = 2^kfx exactly; Q_total <= 2^61 (catches a wrong kfx, a dropped term, a shifted scan)."""
    for P, var in [(1, 1.0), (2, 1.0), (7, 0.1), (1000, 1.0), (4097, 10.0), (65536, 1.0)]:
        x = pfinputs.gaussian_logw(P, var, seed=P)
        st, Q = orc.cumulative(x)
        assert st == 0
        m = int(math.ceil(math.log2(P))) if P > 1 else 0
        k = 61 - m
        assert orc.kfx(P) == k
        q = np.diff(np.concatenate([[0], Q.astype(object)]))
        assert all(int(v) >= 0 for v in q)
        assert int(Q[-1]) <= 2 ** 61
        imax = int(np.argmax(x))
        assert int(q[imax]) == 2 ** k
        lmax = float(np.max(x))
        t = (x.astype(np.float32) - np.float32(lmax)).astype(np.float64)
        exact = np.exp(t) * 2.0 ** k
        qf = np.array([float(v) for v in q])
        # dexp within 2 ulp (2^-23 relative) plus truncation (< 1 unit)
        assert np.all(np.abs(qf - exact) <= exact * 2.0 ** -22 + 1.0)
        # big-int cumulative sum equals Q (u64 never wrapped)
        assert int(sum(int(v) for v in q)) == int(Q[-1])


def test_invalid_inputs(orc):
    """NS-1: NaN, +inf or all -inf -> status 1, identity ancestors, NaN lse."""
    cases = [np.float32([0, np.nan, 1]), np.float32([0, np.inf, 1]), np.full(5, -np.inf, np.float32)]
    for x in cases:
        for s in ("multinomial", "stratified", "systematic", "metropolis"):
            st, a, lse, v, ess = orc.resample(s, x, seed=3, B=4, side=True)
            assert st == 1
            assert list(a) == list(range(len(x)))
            assert math.isnan(lse) and math.isnan(ess)


def test_lse_normw_ess_against_mpmath(orc):
    """NS-13 / P:240-243: lse within 1e-6 of mpmath log-sum-exp of the float inputs;
    normalised weights within 1e-6 of exp(logw - lse); ESS = 1/sum v^2."""
    import mpmath as mp

    for P, var in [(16, 1.0), (1000, 10.0), (5000, 0.1)]:
        x = pfinputs.gaussian_logw(P, var, seed=11)
        st, a, lse, v, ess = orc.resample("systematic", x, seed=1, side=True)
        want = mp.log(mp.fsum(mp.exp(mp.mpf(float(t))) for t in x))
        assert abs(lse - float(want)) <= 1e-6 * max(1.0, abs(float(want)))
        vv = np.exp(x.astype(np.float64) - float(want))
        assert np.all(np.abs(v - vv) <= 1e-6 * np.maximum(vv, 1e-30) + 1e-12)
        ess_exact = 1.0 / float(np.sum(vv * vv))
        assert abs(ess - ess_exact) <= 1e-6 * ess_exact


def test_ess_bands_for_dirichlet(orc):
    """ESS ~ .5P, .1P, .01P for alpha = 1, .1, .01 (Dirichlet weights)."""
    P = 4096
    bands = {1.0: (0.45, 0.55), 0.1: (0.07, 0.12), 0.01: (0.006, 0.016)}
    for alpha, (lo, hi) in bands.items():
        vals = []
        for r in range(8):
            x = pfinputs.dirichlet_logw(P, alpha, seed=100 + r)
            st, a, lse, v, ess = orc.resample("systematic", x, seed=1, side=True)
            vals.append(ess / P)
        assert lo <= float(np.mean(vals)) <= hi, (alpha, np.mean(vals))


# --------------------------------------------------------------------------- conversions
def test_spec_conversion_examples(orc, golden_dir):
    """S:66-77 worked examples and round trip."""
    for line in _lines(os.path.join(golden_dir, "spec_examples.txt")):
        name, inp, out, cite = [s.strip() for s in line.split("|")]
        if name == "offspring_to_ancestors":
            o = np.int32(inp[2:].split(","))
            assert list(orc.offspring_to_ancestors(o)) == [int(v) for v in out[2:].split(",")], cite
        if name == "ancestors_to_offspring":
            a = np.int32(inp[2:].split(","))
            assert list(orc.ancestors_to_offspring(a)) == [int(v) for v in out[2:].split(",")], cite
    rng = np.random.default_rng(5)
    for _ in range(50):
        P = int(rng.integers(1, 40))
        o = rng.multinomial(P, np.ones(P) / P).astype(np.int32)
        assert np.array_equal(orc.ancestors_to_offspring(orc.offspring_to_ancestors(o)), o)


def _weights_case(w):
    with np.errstate(divide="ignore"):
        return np.log(np.float32(w)).astype(np.float32)


def test_spec_resampler_examples(orc):
    """S:152, S:161-162, S:170-171, S:179 (Fig. 1)."""
    # w=[2,1,1], P=3, u=0.3 -> o=[2,0,1]
    st, Q = orc.cumulative(_weights_case([2, 1, 1]))
    a = orc.systematic_from_R(Q, int(0.3 * 2 ** 64))
    assert list(orc.ancestors_to_offspring(a)) == [2, 0, 1]
    for seed in range(20):
        # S:152 single support (multinomial), S:162 (stratified)
        _, a = orc.resample("multinomial", _weights_case([0, 0, 5, 0]), seed)
        assert list(a) == [2, 2, 2, 2]
        _, a = orc.resample("stratified", _weights_case([1, 0, 0, 0]), seed)
        assert list(orc.ancestors_to_offspring(a)) == [4, 0, 0, 0]
        # S:161, S:170 uniform weights
        for s in ("stratified", "systematic"):
            _, a = orc.resample(s, _weights_case([1, 1, 1, 1]), seed)
            assert list(orc.ancestors_to_offspring(a)) == [1, 1, 1, 1]
        # S:179 B = 0 identity
        _, a = orc.resample("metropolis", _weights_case([3, 1, 2, 5]), seed, B=0)
        assert list(a) == [0, 1, 2, 3]


def test_resampling_error_example():
    """the Fig. 2 error metric for P=2, w=[1,1], o=[2,0] is 0.5."""
    o = np.array([2, 0]); v = np.array([0.5, 0.5])
    assert float(np.sum((o / 2 - v) ** 2)) == 0.5


# --------------------------------------------------------------------------- invariants
@pytest.mark.parametrize("scheme", ["multinomial", "stratified", "systematic", "metropolis"])
def test_invariants(orc, scheme):
    """P draws with replacement -> sum o = P, indices in range, zero weights never
    selected by the prefix-sum schemes (G6), sorted schemes give nondecreasing ancestors."""
    for P in (1, 2, 3, 7, 8, 16, 1000, 4097):
        for var in (0.1, 1.0, 10.0):
            x = pfinputs.with_neg_inf_runs(pfinputs.gaussian_logw(P, var, seed=P + int(var * 10)))
            st, a = orc.resample(scheme, x, seed=P * 31 + 7, B=8)
            assert st == 0
            assert a.min() >= 0 and a.max() < P
            assert orc.ancestors_to_offspring(a).sum() == P
            if scheme != "metropolis":
                assert np.all(np.isfinite(x[a]))
            else:  # a chain only moves to positive weights (NS-11 strict compare, R8)
                moved = a != np.arange(P)
                assert np.all(np.isfinite(x[a[moved]]))
            if scheme in ("stratified", "systematic"):
                assert np.all(np.diff(a) >= 0)


def test_uniform_weights_identity(orc):
    """R6/NS-7: all-equal weights, P a power of two -> stratified & systematic give identity."""
    for P in (2, 4, 16, 1024, 65536):
        for s in ("stratified", "systematic"):
            for seed in (1, 2, 3):
                _, a = orc.resample(s, pfinputs.equal_logw(P, -3.5), seed)
                assert np.array_equal(a, np.arange(P))


def test_systematic_floor_ceil(orc):
    """Kitagawa systematic: o_i in {floor(P q_i/Q), ceil(P q_i/Q)} exactly
    (BJ north_star pin; tighter than S:167).  Exact rational arithmetic on the oracle's q."""
    rng = np.random.default_rng(9)
    for trial in range(300):
        P = int(rng.integers(2, 200))
        x = pfinputs.gaussian_logw(P, float(rng.choice([0.1, 1, 10])), seed=trial)
        st, Q = orc.cumulative(x)
        _, a = orc.resample("systematic", x, seed=trial + 1000)
        o = orc.ancestors_to_offspring(a)
        Qi = [int(v) for v in Q]
        q = [Qi[0]] + [Qi[i] - Qi[i - 1] for i in range(1, P)]
        for i in range(P):
            e = Fraction(P * q[i], Qi[-1])
            assert math.floor(e) <= o[i] <= math.ceil(e), (trial, i)


# --------------------------------------------------------------------------- brute force
def _brute(scheme, x, seed, filt=0):
    """Independent big-int re-derivation of the ancestors from the Fig. 1 definitions with a
    linear scan (no binary search, no 128-bit tricks)."""
    P = len(x)
    import oracle as orc_mod

    st, Q = orc_mod.cumulative(x)
    Q = [int(v) for v in Q]
    tot = Q[-1]
    if P == 1:
        return [0]
    D = (1 << (64 - (P - 1).bit_length())) if P & (P - 1) == 0 else ((1 << 64) - 1) // P
    out = []
    for k in range(P):
        if scheme == "multinomial":
            R = phx.half(phx.draw(seed, k >> 1, 0, 1, filt), k & 1)
            pos = R * tot >> 64
        elif scheme == "stratified":
            R = phx.half(phx.draw(seed, k >> 1, 0, 2, filt), k & 1)
            pos = (k * D + (R * D >> 64)) * tot >> 64
        else:
            R = phx.half(phx.draw(seed, 0, 0, 3, filt), 0)
            pos = (k * D + (R * D >> 64)) * tot >> 64
        out.append(next(i for i in range(P) if Q[i] > pos))
    return out


def test_bruteforce_search_small(orc):
    """Linear-scan big-int recomputation equals the oracle (catches mulhi, index, tie errors)."""
    for P in (1, 2, 3, 5, 8, 13, 64):
        for seed in (0, 1, 0xDEADBEEFCAFEF00D):
            x = pfinputs.with_neg_inf_runs(pfinputs.gaussian_logw(P, 1.0, seed=P))
            for s in ("multinomial", "stratified", "systematic"):
                _, a = orc.resample(s, x, seed, filter_index=3)
                assert list(a) == _brute(s, x, seed, 3), (P, seed, s)


def _chi2_sf(stat, dof):
    from scipy.stats import chi2

    return float(chi2.sf(stat, dof))


def _offspring_counts(orc, scheme, x, nseeds, B=0):
    from collections import Counter

    c = Counter()
    for s in range(nseeds):
        _, a = orc.resample(scheme, x, pfinputs.seed_for(s), B=B)
        c[tuple(orc.ancestors_to_offspring(a))] += 1
    return c


def _gof(counts, pmf, n):
    """Chi-square goodness of fit, pooling cells with expected < 5.  Returns p-value."""
    keys = set(pmf) | set(counts)
    for k in counts:
        assert pmf.get(k, 0.0) > 0.0, f"impossible outcome {k}"
    exp_obs = sorted(((pmf.get(k, 0.0) * n, counts.get(k, 0)) for k in keys), reverse=True)
    stat, dof, pe, po = 0.0, 0, 0.0, 0
    for e, o in exp_obs:
        if e >= 5:
            stat += (o - e) ** 2 / e
            dof += 1
        else:
            pe += e; po += o
    if pe > 0:
        stat += (po - pe) ** 2 / max(pe, 1e-12)
        dof += 1
    return _chi2_sf(stat, max(dof - 1, 1))


def _probs(orc, x):
    st, Q = orc.cumulative(x)
    Qi = [int(v) for v in Q]
    q = [Qi[0]] + [Qi[i] - Qi[i - 1] for i in range(1, len(Qi))]
    return [Fraction(v, Qi[-1]) for v in q]


def _pmf_multinomial(p, P):
    from itertools import product

    pmf = {}
    def rec(i, left, cur):
        if i == len(p) - 1:
            o = cur + [left]
            pr = Fraction(math.factorial(P))
            for oi, pi in zip(o, p):
                pr *= pi ** oi / math.factorial(oi)
            if pr > 0:
                pmf[tuple(o)] = float(pr)
            return
        for c in range(left + 1):
            rec(i + 1, left - c, cur + [c])
    rec(0, P, [])
    return pmf


def _pmf_stratified(p, P):
    cum = [Fraction(0)]
    for v in p:
        cum.append(cum[-1] + v)
    dist = {tuple([0] * len(p)): Fraction(1)}
    for k in range(P):
        lo, hi = Fraction(k, P), Fraction(k + 1, P)
        cat = []
        for i in range(len(p)):
            ov = max(Fraction(0), min(hi, cum[i + 1]) - max(lo, cum[i])) * P
            if ov > 0:
                cat.append((i, ov))
        nd = {}
        for o, pr in dist.items():
            for i, pi in cat:
                oo = list(o); oo[i] += 1
                nd[tuple(oo)] = nd.get(tuple(oo), 0) + pr * pi
        dist = nd
    return {k: float(v) for k, v in dist.items()}


def _pmf_systematic(p, P):
    cum = [Fraction(0)]
    for v in p:
        cum.append(cum[-1] + v)
    bps = {Fraction(0), Fraction(1)}
    for c in cum:
        for k in range(P):
            u = P * c - k
            if 0 < u < 1:
                bps.add(u)
    bps = sorted(bps)
    pmf = {}
    for lo, hi in zip(bps[:-1], bps[1:]):
        u = (lo + hi) / 2
        o = [0] * len(p)
        for k in range(P):
            y = (k + u) / P
            i = next(i for i in range(len(p)) if cum[i + 1] > y)
            o[i] += 1
        pmf[tuple(o)] = pmf.get(tuple(o), 0.0) + float(hi - lo)
    return pmf


@pytest.mark.parametrize("scheme,builder", [("multinomial", _pmf_multinomial),
                                            ("stratified", _pmf_stratified),
                                            ("systematic", _pmf_systematic)])
def test_bruteforce_offspring_law(orc, scheme, builder):
    """Brute force at P <= 8: exact pmf of the offspring vector (Fig. 1(a)-(c))
    vs oracle frequencies over many seeds (catches biased positions or a wrong stratum width)."""
    n = 6000
    for P, seed in ((3, 1), (4, 2), (5, 3)):
        x = pfinputs.gaussian_logw(P, 1.0, seed=seed)
        pmf = builder(_probs(orc, x), P)
        assert abs(sum(pmf.values()) - 1) < 1e-12
        counts = _offspring_counts(orc, scheme, x, n)
        assert _gof(counts, pmf, n) > 1e-4, (scheme, P)


def test_unbiasedness_and_closed_form_errors(orc):
    """E[o_i] = P v_i (unbiased schemes) and closed-form mean errors of the Fig. 2 metric
    (P:213-214): multinomial (1 - sum v^2)/P; systematic sum f(1-f)/P^2; stratified
    sum_i sum_k p_ki(1-p_ki)/P^2.  Also the ordering of P:224-226."""
    P, R = 16, 4000
    x = pfinputs.gaussian_logw(P, 1.0, seed=77)
    p = np.array([float(v) for v in _probs(orc, x)])
    cum = np.concatenate([[0], np.cumsum(p)])
    closed = {"multinomial": (1 - np.sum(p * p)) / P}
    f = P * p - np.floor(P * p)
    closed["systematic"] = float(np.sum(f * (1 - f))) / P ** 2
    pk = np.array([[max(0.0, min((k + 1) / P, cum[i + 1]) - max(k / P, cum[i])) * P for i in range(P)]
                   for k in range(P)])
    closed["stratified"] = float(np.sum(pk * (1 - pk))) / P ** 2
    var_o = {"multinomial": P * p * (1 - p), "stratified": np.sum(pk * (1 - pk), axis=0),
             "systematic": None}
    means = {}
    for s in ("multinomial", "stratified", "systematic"):
        O = np.zeros((R, P))
        for r in range(R):
            _, a = orc.resample(s, x, pfinputs.seed_for(r + 500))
            O[r] = orc.ancestors_to_offspring(a)
        err = np.sum((O / P - p) ** 2, axis=1)
        means[s] = err.mean()
        se = err.std(ddof=1) / math.sqrt(R)
        assert abs(err.mean() - closed[s]) <= 5 * se + 1e-12, (s, err.mean(), closed[s])
        mean_o = O.mean(axis=0)
        if var_o[s] is not None:
            z = (mean_o - P * p) / np.sqrt(var_o[s] / R + 1e-300)
            assert np.all(np.abs(z[var_o[s] > 0]) < 5), (s, z)
        else:
            sd = O.std(axis=0, ddof=1) / math.sqrt(R)
            assert np.all(np.abs(mean_o - P * p) <= 5 * sd + 1e-9)
    assert means["stratified"] < means["multinomial"]


# --------------------------------------------------------------------------- Metropolis
def _metro_kernel(w, P):
    """Exact one-step kernel of NS-11: uniform proposal over all indices and
    acceptance on the 24-bit u grid, fl32(u w_k) < w_j counted over all 2^24 grid points."""
    u = (np.arange(1 << 24, dtype=np.float64) * 2.0 ** -24).astype(np.float32)
    K = np.zeros((P, P))
    for k in range(P):
        for j in range(P):
            if j == k:
                continue
            acc = np.count_nonzero((u * np.float32(w[k])) < np.float32(w[j])) / float(1 << 24)
            K[k, j] = acc / P
        K[k, k] = 1.0 - K[k].sum()
    return K


def test_metropolis_exact_small(orc):
    """P <= 4 brute force: each chain's ancestor law equals row i of K^B (NS-11); catches a wrong
    proposal map, a flipped comparison or a reused random word."""
    n = 20000
    for P, B, seed in ((3, 1, 4), (3, 5, 5), (4, 3, 6)):
        x = pfinputs.gaussian_logw(P, 1.0, seed=seed)
        st, w = orc.weights(x)
        KB = np.linalg.matrix_power(_metro_kernel(w, P), B)
        counts = np.zeros((P, P))
        for s in range(n):
            _, a = orc.resample("metropolis", x, pfinputs.seed_for(s), B=B)
            counts[np.arange(P), a] += 1
        for i in range(P):
            e = KB[i] * n
            stat = float(np.sum((counts[i] - e) ** 2 / np.maximum(e, 1e-12)))
            assert _chi2_sf(stat, P - 1) > 1e-4, (P, B, i, counts[i], e)


def _corrected_T_power(alpha, beta, l):
    """Eq. (3) with the stationary term corrected (R11), states ordered (Z=1, Z=0)."""
    lam = 1 - alpha - beta
    s = alpha + beta
    return (np.array([[beta, alpha], [beta, alpha]]) + lam ** l * np.array([[alpha, -alpha], [-beta, beta]])) / s


def test_eq3_corrected_form():
    """R11: the corrected Eq. (3) satisfies T^0 = I, T^1 = T (Eq. 1) and T^l = matrix power;
    the printed form fails T^0 = I."""
    rng = np.random.default_rng(3)
    for _ in range(100):
        a, b = rng.uniform(0, 0.5, 2)
        T = np.array([[1 - a, a], [b, 1 - b]])
        assert np.allclose(_corrected_T_power(a, b, 0), np.eye(2), atol=1e-12)
        l = int(rng.integers(1, 50))
        assert np.allclose(_corrected_T_power(a, b, l), np.linalg.matrix_power(T, l), atol=1e-10)
        printed0 = (np.array([[a, b], [a, b]]) + np.array([[a, -a], [-b, b]])) / (a + b)
        assert not np.allclose(printed0, np.eye(2))


def test_metropolis_max_particle_closed_form(orc):
    """exact lumping of the max particle (beta = 1/P, alpha of Eq. (2)); the mean count
    of chains ending on p_max follows the corrected Eq. (3) at every B (catches a missing
    'always accept the max' or a wrong chain start)."""
    P, R = 64, 400
    x = pfinputs.gaussian_logw(P, 1.0, seed=21)
    st, w = orc.weights(x)
    imax = int(np.argmax(w))
    v = w.astype(np.float64) / w.astype(np.float64).sum()
    wmax = v[imax]
    beta = 1.0 / P
    alpha = float(np.sum(np.delete(v, imax))) / (P * wmax)  # Eq. (2)
    for B in (1, 4, 16, 64, 256):
        T = _corrected_T_power(alpha, beta, B)
        expect = T[0, 0] + (P - 1) * T[1, 0]
        pvar = T[0, 0] * (1 - T[0, 0]) + (P - 1) * T[1, 0] * (1 - T[1, 0])
        cnt = []
        for r in range(R):
            _, a = orc.resample("metropolis", x, pfinputs.seed_for(10000 + r), B=B)
            cnt.append(np.count_nonzero(a == imax))
        se = math.sqrt(pvar / R)
        assert abs(np.mean(cnt) - expect) < 5 * se, (B, np.mean(cnt), expect)


def test_metropolis_converges_to_multinomial(orc):
    """Metropolis converges to multinomial as B grows; with B from Eq. (5) at eps=.01
    (scaled 4x) the ancestor law of every chain matches v (chi-square), and the Fig. 2 error
    approaches (1 - sum v^2)/P."""
    P, R = 32, 600
    x = pfinputs.gaussian_logw(P, 0.1, seed=8)
    st, w = orc.weights(x)
    v = w.astype(np.float64) / w.astype(np.float64).sum()
    B = 4 * orc.required_B(P, float(v.max()), 0.01)
    counts = np.zeros(P)
    errs = []
    for r in range(R):
        _, a = orc.resample("metropolis", x, pfinputs.seed_for(20000 + r), B=B)
        o = orc.ancestors_to_offspring(a)
        counts += o
        errs.append(np.sum((o / P - v) ** 2))
    e = v * P * R
    stat = float(np.sum((counts - e) ** 2 / e))
    assert _chi2_sf(stat, P - 1) > 1e-4
    closed = (1 - np.sum(v * v)) / P
    se = np.std(errs, ddof=1) / math.sqrt(R)
    assert abs(np.mean(errs) - closed) < 5 * se


def test_metropolis_single_support(orc):
    """R8: chains off the support move only onto it, with probability 1-(1-1/P)^B."""
    P, B, R = 8, 5, 3000
    x = pfinputs.single_support_logw(P, 5)
    hits = 0
    for r in range(R):
        _, a = orc.resample("metropolis", x, pfinputs.seed_for(r), B=B)
        assert np.all((a == 5) | (a == np.arange(P)))
        hits += np.count_nonzero(a[np.arange(P) != 5] == 5)
    p = 1 - (1 - 1 / P) ** B
    n = R * (P - 1)
    assert abs(hits / n - p) < 5 * math.sqrt(p * (1 - p) / n)


def test_required_B_golden(orc, golden_dir):
    """Eq. (5) against mpmath values (tests/golden/make_eq5.py)."""
    for line in _lines(os.path.join(golden_dir, "eq5_required_B.txt")):
        P, w, e, B = line.split()
        assert orc.required_B(int(P), float(w), float(e)) == int(B), line


# --------------------------------------------------------------------------- permute / gather
def test_permute_postconditions(orc):
    """NS-15: permutation of the ancestor multiset; a'_i = i iff o_i > 0; the free slots, in
    ascending order, hold the extra copies in ascending survivor order (unique given o)."""
    rng = np.random.default_rng(4)
    for trial in range(200):
        P = int(rng.integers(1, 300))
        x = pfinputs.gaussian_logw(P, float(rng.choice([0.1, 1, 10])), seed=trial)
        _, a = orc.resample(["multinomial", "stratified", "systematic"][trial % 3], x, trial)
        a = rng.permutation(a).astype(np.int32)  # any input order
        perm = orc.permute(a)
        o = np.bincount(a, minlength=P)
        assert np.array_equal(np.sort(perm), np.sort(a))
        surv = o > 0
        assert np.array_equal(perm[surv], np.nonzero(surv)[0])
        free_vals = perm[~surv]
        assert np.all(np.diff(free_vals) >= 0)
        assert np.all(o[free_vals] > 1)


def test_gather(orc):
    """NS-16: in-place gather with the canonical permutation equals the out-of-place
    gather X[perm] (numpy fancy indexing) and X[anc] up to the row order of copies."""
    rng = np.random.default_rng(6)
    for P, D in ((1, 1), (17, 16), (300, 3)):
        x = pfinputs.gaussian_logw(P, 1.0, seed=P)
        _, a = orc.resample("multinomial", x, 12)
        X = pfinputs.state_matrix(P, D, seed=P)
        perm = orc.permute(a)
        Y = orc.gather_inplace(X, perm)
        assert np.array_equal(Y, X[perm])
        Z = orc.gather_out(X, a)
        assert np.array_equal(Z, X[a])
        assert sorted(map(tuple, Y.tolist())) == sorted(map(tuple, Z.tolist()))


def test_batched_matches_single(orc):
    """R-batched: filter n of a batch equals a single call with filter_index first+n."""
    N, P = 5, 100
    x = pfinputs.gaussian_logw(P, 1.0, seed=3, N=N)
    for s in ("multinomial", "stratified", "systematic", "metropolis"):
        st, A = orc.resample_batched(s, x, 99, B=6, first_filter=40)
        for n in range(N):
            _, a = orc.resample(s, x[n], 99, B=6, filter_index=40 + n)
            assert np.array_equal(A[n], a)
        # different filters draw different streams
        if s != "metropolis":
            assert not all(np.array_equal(A[0], A[n]) for n in range(1, N)) or s == "systematic"


# --------------------------------------------------------------------------- NS-12 (a6)
def test_dlog_accuracy(orc):
    """NS-12: the deterministic double log is within 2 ulp of math.log on (0, 1] (catches a wrong
    series coefficient, a dropped ln2 term or a wrong sqrt(2) reduction)."""
    rng = np.random.default_rng(0)
    xs = np.concatenate([(rng.integers(0, 2 ** 32, 50000) + 0.5) / 2 ** 32,
                         [2 ** -33, 0.5, 0.7071067811865476, 0.7071067811865475, 1 - 2 ** -33, 0.999999]])
    for x in xs:
        d, e = orc.dlog(float(x)), math.log(float(x))
        assert abs(d - e) <= 2 * math.ulp(e), x
    assert orc.dlog(1.0) == 0.0


def test_spacings_are_uniform_order_statistics(orc):
    """NS-12: e_k >= 1 with mean 2^24 (Exp(1) in 2^-24 units), G strictly increasing, and
    E[G_k / G_P] = (k+1)/(P+1) (the k-th of P uniform order statistics)."""
    P, R = 9, 3000
    ratios = np.zeros((R, P))
    e_all = []
    for r in range(R):
        G = orc.spacings(P, pfinputs.seed_for(r), filter_index=r % 7).astype(np.float64)
        assert np.all(np.diff(G) >= 1) and G[0] >= 1
        e_all.append(np.diff(np.concatenate([[0.0], G])))
        ratios[r] = G[:P] / G[P]
    e_all = np.concatenate(e_all) / 2.0 ** 24
    assert abs(e_all.mean() - 1.0) < 5 * 1.0 / math.sqrt(len(e_all))
    k = np.arange(P)
    mean = (k + 1) / (P + 1)
    var = mean * (1 - mean) / (P + 2)  # Beta(k+1, P-k) variance
    z = (ratios.mean(axis=0) - mean) / np.sqrt(var / R)
    assert np.all(np.abs(z) < 5), z


def test_sorted_multinomial_search_and_invariants(orc):
    """a6: big-int recomputation of x_k = floor(G_k Q / G_P) and linear-scan search equal the oracle;
    ancestors nondecreasing; zero weights never chosen."""
    for P in (1, 2, 5, 64, 1000):
        x = pfinputs.with_neg_inf_runs(pfinputs.gaussian_logw(P, 1.0, seed=P))
        for seed in (3, 0xABCDEF0123456789):
            st, a = orc.resample_sorted_multinomial(x, seed, filter_index=2)
            _, Q = orc.cumulative(x)
            Q = [int(v) for v in Q]
            G = [int(v) for v in orc.spacings(P, seed, 2)]
            want = [next(i for i in range(P) if Q[i] > G[k] * Q[-1] // G[P]) for k in range(P)]
            assert list(a) == want
            assert np.all(np.diff(a) >= 0) and np.all(np.isfinite(x[a]))


def test_sorted_multinomial_offspring_law(orc):
    """a6 has the multinomial law (Fig. 1(a)): exact multinomial pmf of the offspring
    vector at P <= 5 vs oracle frequencies (chi-square)."""
    from collections import Counter

    n = 6000
    for P, seed in ((3, 1), (4, 2), (5, 3)):
        x = pfinputs.gaussian_logw(P, 1.0, seed=seed)
        pmf = _pmf_multinomial(_probs(orc, x), P)
        c = Counter()
        for s in range(n):
            _, a = orc.resample_sorted_multinomial(x, pfinputs.seed_for(s))
            c[tuple(orc.ancestors_to_offspring(a))] += 1
        assert _gof(c, pmf, n) > 1e-4, P


def test_kalman_oracle_against_joint_gaussian():
    """C4 oracle (R-20): the Kalman log-likelihood equals the exact joint Gaussian log-density of
    y_1:T (stationary AR(1) covariance phi^|s-t| sigma_x^2/(1-phi^2) + sigma_y^2 delta_st)."""
    from scipy.stats import multivariate_normal

    from oracle.kalman import kalman_loglik

    for phi, sx, sy, T in ((0.9, 1.0, 1.0, 30), (0.5, 0.7, 2.0, 12)):
        ys = pfinputs.lg_observations(T, phi, sx, sy, seed=T)
        ll, _ = kalman_loglik(ys, phi, sx, sy)
        s0 = sx * sx / (1 - phi * phi)
        idx = np.arange(T)
        C = s0 * phi ** np.abs(idx[:, None] - idx[None, :]) + sy * sy * np.eye(T)
        want = multivariate_normal(mean=np.zeros(T), cov=C).logpdf(ys)
        assert abs(ll - want) < 1e-9 * max(1.0, abs(want)), (ll, want)


# --------------------------------------------------------------------------- NS-3d (R-21)
@pytest.mark.parametrize("c", [0.0, 2.0 ** 30, -(2.0 ** 40)])
def test_f64_exact_shift_reduces_to_f32(orc, c):
    """NS-3d: resampling depends on the log-weights only through logw_i - max, so
    binary64 inputs x + c with an EXACT shift c give the float32 path's ancestors on x, and
    lse(x + c) = lse(x) + c.  Catches rounding logw or lmax to float before subtracting
    (x + 2^30 in float32 keeps only multiples of 64), a float max, and a dropped lmax in lse."""
    for P, seed in [(1, 1), (16, 2), (1000, 3), (4097, 4)]:
        x = pfinputs.grid_logw(P, 4.0, seed=seed)
        x64 = x.astype(np.float64) + c
        assert np.all(x64 - c == x.astype(np.float64))  # the shift is exact
        for s in ("multinomial", "stratified", "systematic", "metropolis"):
            st, a, lse, v, ess = orc.resample_f64(s, x64, seed=seed, B=9, side=True)
            st2, a2, lse2, v2, ess2 = orc.resample(s, x, seed=seed, B=9, side=True)
            assert st == st2 == 0
            assert np.array_equal(a, a2), s
            assert np.array_equal(v, v2) and ess == ess2
            assert abs(lse - (lse2 + c)) <= 1e-12 * max(1.0, abs(c))
        st, a = orc.resample_f64("multinomial", x64, seed=seed, sorted=True)
        assert np.array_equal(a, orc.resample_sorted_multinomial(x, seed)[1])


def test_f64_large_offset_against_logsumexp(orc):
    """NS-3d / NS-13 at an inexact offset (-1e7, where float32 log-weights would keep only
    multiples of 1): lse - offset against the fp64 log-sum-exp, normalised weights against
    exp(logw - lse) (numpy fp64), and a float32 path that ignores the offset would fail it."""
    for P, var in [(16, 1.0), (1000, 10.0), (3000, 0.1)]:
        x = pfinputs.gaussian_logw_f64(P, var, offset=-1e7, seed=P)
        st, a, lse, v, ess = orc.resample_f64("stratified", x, seed=5, side=True)
        assert st == 0
        m = float(np.max(x))
        want = m + math.log(float(np.sum(np.exp(x - m))))
        assert abs((lse + 1e7) - (want + 1e7)) <= 1e-5
        vv = np.exp(x - want)
        assert np.all(np.abs(v - vv) <= 2e-6 * vv + 1e-12)
        ess_exact = 1.0 / float(np.sum(vv * vv))
        assert abs(ess - ess_exact) <= 1e-5 * ess_exact
        # the offspring track P * v within one (stratified)
        o = orc.ancestors_to_offspring(a)
        assert np.all(np.abs(o - P * vv) < 2.0 + 1e-9)


def test_f64_invalid_and_zero_weights(orc):
    """NS-1 on the doubles: NaN, +inf, all -inf -> status 1, identity, NaN lse.  Entries more
    than 88 below the maximum (down to -1e300, beyond float range) weigh zero (NS-4 step 1)
    and are never selected; a lone finite entry takes every slot."""
    bad = [np.array([0.0, np.nan, 1.0]), np.array([0.0, np.inf]), np.full(4, -np.inf)]
    for x in bad:
        for s in ("multinomial", "stratified", "systematic", "metropolis"):
            st, a, lse, v, ess = orc.resample_f64(s, x, seed=3, B=4, side=True)
            assert st == 1 and list(a) == list(range(len(x))) and math.isnan(lse)
    x = np.array([-1e300, 5.0e8, 5.0e8 - 100.0, -np.inf, 5.0e8 - 1.0, 5.0e8 - 3e38])
    for s in ("multinomial", "stratified", "systematic", "metropolis"):
        st, a = orc.resample_f64(s, x, seed=7, B=200)
        assert st == 0 and set(a.tolist()) <= {1, 4}
    x = np.array([-np.inf, -1e300, 12345.678, -np.inf])
    for s in ("multinomial", "stratified", "systematic", "metropolis"):
        st, a, lse, v, ess = orc.resample_f64(s, x, seed=8, B=200, side=True)  # (3/4)^200 to stay at a zero weight
        assert st == 0 and list(a) == [2, 2, 2, 2]
        assert lse == 12345.678 and list(v) == [0.0, 0.0, 1.0, 0.0] and ess == 1.0


# --------------------------------------------------------------------------- NS-17 (R-14)
SORTED_SCHEMES = ("multinomial", "stratified", "systematic")


def test_sorted_weights_bruteforce(orc):
    """NS-17: the paper's 'sorting enabled' series: an independent re-derivation:
    Python's stable sort by (-logw, index) (so +0 == -0 and ties keep index order), the
    linear-scan big-int ancestors of the sorted weights, mapped back through sigma.  Catches
    an ascending sort, unstable ties, and mapping with sigma^-1 instead of sigma."""
    rng = np.random.default_rng(17)
    for trial in range(60):
        P = int(rng.integers(1, 40))
        x = pfinputs.gaussian_logw(P, float(rng.choice([0.1, 1, 10])), seed=trial)
        if trial % 3 == 0:  # ties, signed zeros and zero weights
            x = np.round(x).astype(np.float32)
            x[x == 0] = np.float32(-0.0) if trial % 2 else np.float32(0.0)
            x[:: max(1, P // 3)] = -np.inf
            if not np.any(np.isfinite(x)):
                x[0] = 0.0
        sigma = sorted(range(P), key=lambda i: (-float(x[i]), i))
        y = np.ascontiguousarray(x[sigma])
        for s in SORTED_SCHEMES:
            seed = 1000 + trial
            st, a = orc.resample_sorted_weights(s, x, seed)
            assert st == 0
            assert [int(v) for v in a] == [sigma[b] for b in _brute(s, y, seed)], (trial, s)


def test_sorted_weights_rotation_and_side_outputs(orc):
    """Distinct descending y rotated by r: sigma(j) = (j + r) mod P, so a_k = (b_k + r) mod P
    with b the plain ancestors of y; v_x[i] = v_y[(i - r) mod P]; lse and ESS unchanged.
    Already-sorted input (r = 0) is the plain resampler."""
    for P, r in [(5, 0), (100, 1), (4097, 1234)]:
        y = np.sort(pfinputs.gaussian_logw(P, 1.0, seed=P))[::-1].copy()
        assert np.all(np.diff(y) < 0)  # distinct, descending
        x = np.roll(y, r)
        for s in SORTED_SCHEMES:
            st, a, lse, v, ess = orc.resample_sorted_weights(s, x, 77, side=True)
            _, b, lse_y, v_y, ess_y = orc.resample(s, y, 77, side=True)
            assert np.array_equal(a, (b + r) % P)
            assert np.array_equal(v, np.roll(v_y, r))
            assert lse == lse_y and ess == ess_y


def test_sorted_weights_laws(orc):
    """Sorting changes which uniforms land on which particle, not the per-particle law:
    systematic o_i in {floor(P q_i/Q), ceil(P q_i/Q)} exactly; multinomial and stratified
    unbiased (E[o_i] = P v_i, z-test over seeds); invalid filters give the identity."""
    for trial in range(100):
        P = 2 + trial % 150
        x = pfinputs.gaussian_logw(P, 4.0, seed=trial)
        st, Q = orc.cumulative(x)
        Qi = [int(v) for v in Q]
        q = [Qi[0]] + [Qi[i] - Qi[i - 1] for i in range(1, P)]
        o = orc.ancestors_to_offspring(orc.resample_sorted_weights("systematic", x, trial)[1])
        for i in range(P):
            e = Fraction(P * q[i], Qi[-1])
            assert math.floor(e) <= o[i] <= math.ceil(e), (trial, i)
    P, R = 50, 3000
    x = pfinputs.gaussian_logw(P, 2.0, seed=5)
    _, _, _, v, _ = orc.resample("systematic", x, 1, side=True)
    for s in ("multinomial", "stratified"):
        tot = np.zeros(P)
        tot2 = np.zeros(P)
        for r in range(R):
            o = orc.ancestors_to_offspring(orc.resample_sorted_weights(s, x, pfinputs.seed_for(r))[1]).astype(float)
            tot += o
            tot2 += o * o
        mean = tot / R
        var = np.maximum(tot2 / R - mean * mean, 1e-12)
        z = (mean - P * v.astype(float)) / np.sqrt(var / R)
        assert np.max(np.abs(z)) < 4.5, s
    for bad in (np.float32([0, np.nan, 1]), np.full(3, -np.inf, np.float32)):
        for s in SORTED_SCHEMES:
            st, a = orc.resample_sorted_weights(s, bad, 3)
            assert st == 1 and list(a) == [0, 1, 2]


# --------------------------------------------------------------------------- C4 model (NS-18)
def test_lg_model_noise_is_standard_normal(orc):
    """oracle/lg_model.py: the Box-Muller noise of the C4 step is N(0, 1) (KS test against the
    normal CDF over 4 x 4096 draws; pairs uncorrelated), and one step of the AR(1) from x has mean
    phi x and variance sigma_x^2 per dimension (R-20), the weight the Gaussian log-density."""
    from scipy import stats

    from oracle import lg_model

    z = np.concatenate([lg_model.noise(i, 3, 6, 12345) for i in range(4096)])
    assert stats.kstest(z, "norm").pvalue > 1e-3
    zz = z.reshape(-1, 4)
    assert abs(np.corrcoef(zz[:, 0], zz[:, 1])[0, 1]) < 0.05
    assert abs(np.corrcoef(zz[:, 0], zz[:, 2])[0, 1]) < 0.05
    P, D, phi, sx, sy = 4000, 5, 0.9, 0.7, 1.3
    X = np.full((P, D), 2.0)
    Xn, logw = lg_model.lg_step(X, 0.4, 7, phi, sx, sy, 99)
    d = Xn - phi * X
    se = sx / math.sqrt(P)
    assert np.all(np.abs(d.mean(axis=0)) < 5 * se)
    assert np.all(np.abs(d.std(axis=0) / sx - 1.0) < 0.06)
    assert np.allclose(logw, -((0.4 - Xn[:, 0]) ** 2) / (2 * sy * sy))
    # distinct time steps and particles draw distinct noise (the Philox counter layout)
    assert not np.allclose(lg_model.noise(5, 1, 6, 99), lg_model.noise(5, 2, 6, 99))
    X0 = lg_model.lg_init(3000, 4, phi, sx, 7)
    assert abs(X0.var() / (sx * sx / (1 - phi * phi)) - 1.0) < 0.06
