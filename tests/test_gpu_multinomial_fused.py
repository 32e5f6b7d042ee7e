"""GPU parity of the multinomial's one-launch search structure (the cluster kernel's bucket
mode: Q, totals, status, side outputs and the bucket index in one launch, then the per-slot
searches) against the oracle, for filters of 4097..65536 particles (power-of-two and not): batches with
invalid filters, -inf runs, side outputs, status, offspring and an explicit workspace; the
multi-launch path (PF_NO_FUSION) gives the same ancestors."""
from __future__ import annotations

import math

import numpy as np
import pytest

import pfinputs

pytestmark = pytest.mark.gpu


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


@pytest.mark.parametrize("N,P", [(1, 8192), (40, 16384), (300, 8192), (7, 65536), (1, 65536), (1, 4097),
                                 (20, 12289), (9, 50001), (200, 40000), (300, 3000), (200, 4096)])
def test_multinomial_bucket_mode(pf, dev, orc, N, P):
    import torch

    x = pfinputs.with_neg_inf_runs(pfinputs.gaussian_logw(P, 4.0, seed=N * 7 + P, N=N))
    if N >= 3:
        x[1, :] = -np.inf
        x[2, P // 2] = np.nan
    g = torch.from_numpy(x).to(dev)
    st = torch.empty(N, dtype=torch.int32, device=dev)
    lse = torch.empty(N, dtype=torch.float64, device=dev)
    ess = torch.empty(N, dtype=torch.float64, device=dev)
    off = torch.empty((N, P), dtype=torch.int32, device=dev)
    v = torch.empty((N, P), dtype=torch.float32, device=dev)
    ws = torch.empty(pf.pf_workspace_bytes("multinomial", N, P) // 4 + 64, dtype=torch.int32, device=dev)
    a = pf.pf_resample_batched("multinomial", g, 99, first_filter=3, status_out=st, lse_out=lse, ess_out=ess,
                               offspring_out=off, normw_out=v, workspace=ws)
    a2 = pf.pf_resample_batched("multinomial", g, 99, first_filter=3, flags=pf.PF_NO_FUSION)
    torch.cuda.synchronize()
    a, st, lse, ess, off, v = (t.cpu().numpy() for t in (a, st, lse, ess, off, v))
    assert np.array_equal(a, a2.cpu().numpy())
    for n in range(N):
        wst, want, wlse, wv, wess = orc.resample("multinomial", x[n], 99, filter_index=3 + n, side=True)
        assert st[n] == wst
        assert np.array_equal(a[n], want), (N, P, n)
        assert np.array_equal(off[n], orc.ancestors_to_offspring(want))
        if wst == 0:
            assert abs(lse[n] - wlse) <= 1e-6 * max(1.0, abs(wlse))
            assert abs(ess[n] - wess) <= 1e-6 * wess
            assert np.all(np.abs(v[n] - wv) <= 1e-6 * np.maximum(np.abs(wv), 1e-30))
        else:
            assert math.isnan(lse[n])


@pytest.mark.parametrize("P", [65537, 1 << 18, (1 << 20) + 3, 1 << 22])
def test_multinomial_cooperative_bucket_mode(pf, dev, orc, P):
    """Single large filters: the cooperative kernel's bucket mode (Q, totals, status, lse / ESS
    and the bucket index in one launch) + the per-slot searches; an all -inf filter and a NaN."""
    import torch

    for case in ("ok", "neg_inf", "nan"):
        x = pfinputs.with_neg_inf_runs(pfinputs.gaussian_logw(P, 2.0, seed=P))
        if case == "neg_inf":
            x[:] = -np.inf
        elif case == "nan":
            x[P // 3] = np.nan
        g = torch.from_numpy(x).to(dev)
        st = torch.empty(1, dtype=torch.int32, device=dev)
        lse = torch.empty(1, dtype=torch.float64, device=dev)
        ess = torch.empty(1, dtype=torch.float64, device=dev)
        off = torch.empty(P, dtype=torch.int32, device=dev)
        a = pf.pf_resample_ex("multinomial", g, 5, filter_index=9, status_out=st, lse_out=lse, ess_out=ess,
                              offspring_out=off)
        a2 = pf.pf_resample_ex("multinomial", g, 5, filter_index=9, flags=pf.PF_NO_FUSION)
        torch.cuda.synchronize()
        wst, want, wlse, _, wess = orc.resample("multinomial", x, 5, filter_index=9, side=True)
        assert int(st.item()) == wst
        assert np.array_equal(a.cpu().numpy(), want), (P, case)
        assert np.array_equal(a2.cpu().numpy(), want)
        assert np.array_equal(off.cpu().numpy(), orc.ancestors_to_offspring(want))
        if wst == 0:
            assert abs(lse.item() - wlse) <= 1e-6 * max(1.0, abs(wlse))
            assert abs(ess.item() - wess) <= 1e-6 * wess
        else:
            assert math.isnan(lse.item())
