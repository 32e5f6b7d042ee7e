"""GPU parity of the pre-sorted weight series (PF_SORT_WEIGHTS, NS-17; the paper's
'sorting enabled' runs) against the oracle's resample_sorted_weights: ancestors,
offspring, permutations and gathered states bit-exact, side outputs within NS-13's 1e-6, over
single filters (one and many radix tiles, ragged tails), batches with strides, ties / signed
zeros / -inf, invalid filters, binary64 input, and both the fused and multi-launch paths."""
from __future__ import annotations

import math

import numpy as np
import pytest

import pfinputs

pytestmark = pytest.mark.gpu

SCHEMES = ["multinomial", "stratified", "systematic"]


@pytest.fixture(scope="module")
def pf():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_1202_6163_b200 import _build

    _build.build()
    import paper_1202_6163_b200 as pf

    return pf


@pytest.fixture(scope="module")
def dev():
    import torch

    return torch.device("cuda:0")


def _gpu(x, dev):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


def _ties(x):
    y = np.round(x * 2).astype(np.float32) / 2
    y[y == 0] = np.float32(-0.0)
    y[::7] = -np.inf
    return y


@pytest.mark.parametrize("scheme", SCHEMES)
def test_sorted_weights_single(pf, dev, orc, scheme):
    import torch

    for P in (1, 2, 3, 16, 1000, 4096, 4097, 12289, 65536, 100003, (1 << 20) + 7):
        for var, tie in ((1.0, False), (10.0, False), (1.0, True)):
            x = pfinputs.gaussian_logw(P, var, seed=P)
            if tie:
                x = _ties(x)
                if not np.any(np.isfinite(x)):
                    x[0] = 0.0
            lse = torch.empty(1, dtype=torch.float64, device=dev)
            ess = torch.empty(1, dtype=torch.float64, device=dev)
            v = torch.empty(P, dtype=torch.float32, device=dev)
            st = torch.empty(1, dtype=torch.int32, device=dev)
            a = pf.pf_resample_ex(scheme, _gpu(x, dev), 21, filter_index=3, lse_out=lse, ess_out=ess, normw_out=v,
                                  status_out=st, flags=pf.PF_SORT_WEIGHTS)
            torch.cuda.synchronize()
            wst, want, wlse, wv, wess = orc.resample_sorted_weights(scheme, x, 21, filter_index=3, side=True)
            assert int(st.item()) == wst == 0
            assert np.array_equal(a.cpu().numpy(), want), (scheme, P, var, tie)
            assert abs(lse.item() - wlse) <= 1e-6 * max(1.0, abs(wlse))
            assert abs(ess.item() - wess) <= 1e-6 * wess
            assert np.all(np.abs(v.cpu().numpy() - wv) <= 1e-6 * np.maximum(np.abs(wv), 1e-30))


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("fusion", [True, False])
def test_sorted_weights_batched(pf, dev, orc, scheme, fusion):
    import torch

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    pf.pf_set_fusion(fusion)
    try:
        for N, P, ld in ((300, 200, 203), (2 * sms, 8192, 8193), (3, 70000, 70001)):
            x = pfinputs.gaussian_logw(ld, 2.0, seed=N + P, N=N)
            x[1] = _ties(x[1])
            x[0, P // 3] = np.nan
            x[N - 1, :] = -np.inf
            st = torch.empty(N, dtype=torch.int32, device=dev)
            off = torch.empty((N, P), dtype=torch.int32, device=dev)
            a = pf.pf_resample_batched(scheme, _gpu(x, dev)[:, :P], 5, first_filter=11, status_out=st,
                                       offspring_out=off, flags=pf.PF_SORT_WEIGHTS)
            torch.cuda.synchronize()
            a, st, off = a.cpu().numpy(), st.cpu().numpy(), off.cpu().numpy()
            for n in range(N):
                wst, want = orc.resample_sorted_weights(scheme, np.ascontiguousarray(x[n, :P]), 5, filter_index=11 + n)
                assert st[n] == wst
                assert np.array_equal(a[n], want), (scheme, N, P, n)
                assert np.array_equal(off[n], orc.ancestors_to_offspring(want))
    finally:
        pf.pf_set_fusion(True)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_sorted_weights_permutation_state_f64(pf, dev, orc, scheme):
    """permuted_out and the in-place state gather on the mapped ancestors; binary64 input
    through the same flag (NS-3d then NS-17)."""
    import torch

    N, P = 20, 5000
    x = pfinputs.gaussian_logw(P, 1.0, seed=9, N=N)
    X = np.stack([pfinputs.state_matrix(P, 8, seed=n) for n in range(N)])
    gX = _gpu(X, dev)
    perm = torch.empty((N, P), dtype=torch.int32, device=dev)
    a = pf.pf_resample_batched(scheme, _gpu(x, dev), 8, permuted_out=perm, state=gX, flags=pf.PF_SORT_WEIGHTS)
    torch.cuda.synchronize()
    a, perm, gX = a.cpu().numpy(), perm.cpu().numpy(), gX.cpu().numpy()
    for n in range(N):
        _, want = orc.resample_sorted_weights(scheme, x[n], 8, filter_index=n)
        assert np.array_equal(a[n], want)
        wp = orc.permute(want)
        assert np.array_equal(perm[n], wp)
        assert np.array_equal(gX[n], orc.gather_inplace(X[n], wp))
    x64 = pfinputs.gaussian_logw_f64(4097, 1.0, offset=-1e7, seed=3)
    a = pf.pf_resample_ex(scheme, _gpu(x64, dev), 4, flags=pf.PF_SORT_WEIGHTS)
    torch.cuda.synchronize()
    _, t, _ = orc.shift_f64(x64)
    assert np.array_equal(a.cpu().numpy(), orc.resample_sorted_weights(scheme, t, 4)[1])


def test_sorted_weights_unsupported(pf, dev):
    import torch

    x = _gpu(pfinputs.gaussian_logw(100, 1.0), dev)
    for scheme, flags in (("metropolis", pf.PF_SORT_WEIGHTS), ("multinomial", pf.PF_SORT_WEIGHTS | pf.PF_SORTED)):
        with pytest.raises(pf.PfError):
            pf.pf_resample_ex(scheme, x, 1, 4, flags=flags)
    torch.cuda.synchronize()
