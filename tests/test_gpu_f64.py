"""GPU parity of the binary64 entry points (pf_resample_ex_f64 / pf_resample_batched_f64,
DESIGN.md NS-3d / R-21) against the CPU oracle's resample_f64 on the same seeded inputs:
ancestors, offspring, permutations and gathered states bit-exact; lse / ess / normalised
weights within NS-13's 1e-6.  Inputs carry the large common offset (-1e7, an accumulated
log-likelihood) the entry points exist for, across every dispatch path of the float path
(warp-per-filter, CTA-per-filter, cluster, cooperative, multi-launch)."""
from __future__ import annotations

import math

import numpy as np
import pytest

import pfinputs

pytestmark = pytest.mark.gpu

SCHEMES = ["multinomial", "stratified", "systematic", "metropolis"]


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


@pytest.mark.parametrize("scheme", SCHEMES + ["sorted"])
@pytest.mark.parametrize("var", [0.1, 1.0, 10.0])
def test_f64_single_filter(pf, dev, orc, scheme, var):
    import torch

    name = "multinomial" if scheme == "sorted" else scheme
    flags = pf.PF_SORTED if scheme == "sorted" else 0
    for P in (1, 2, 7, 16, 1000, 4097, 12289, 65536, 100003, (1 << 20) + 5):
        if scheme == "metropolis" and P > 100003:
            continue
        x = pfinputs.gaussian_logw_f64(P, var, offset=-1e7, seed=P + 1)
        lse = torch.empty(1, dtype=torch.float64, device=dev)
        ess = torch.empty(1, dtype=torch.float64, device=dev)
        v = torch.empty(P, dtype=torch.float32, device=dev)
        st = torch.empty(1, dtype=torch.int32, device=dev)
        a = pf.pf_resample_ex(name, _gpu(x, dev), 31, 16, filter_index=5, lse_out=lse, ess_out=ess, normw_out=v,
                              status_out=st, flags=flags)
        torch.cuda.synchronize()
        wst, want, wlse, wv, wess = orc.resample_f64(name, x, 31, B=16, filter_index=5, side=True,
                                                     sorted=scheme == "sorted")
        assert int(st.item()) == wst == 0
        assert np.array_equal(a.cpu().numpy(), want), (scheme, P)
        # same binary64 maximum on both sides: lse differs only by ln S's summation order
        assert abs(lse.item() - wlse) <= 1e-6
        assert abs(ess.item() - wess) <= 1e-6 * wess
        assert np.all(np.abs(v.cpu().numpy() - wv) <= 1e-6 * np.maximum(np.abs(wv), 1e-30))


@pytest.mark.parametrize("scheme", SCHEMES)
def test_f64_exact_shift_equals_f32_path(pf, dev, orc, scheme):
    """x + 2^30 in binary64 (exact) resamples like x in float32 on the GPU too."""
    import torch

    for P in (16, 4097, 65536):
        x = pfinputs.grid_logw(P, 4.0, seed=P)
        a32 = pf.pf_resample_ex(scheme, _gpu(x, dev), 3, 12)
        a64 = pf.pf_resample_ex(scheme, _gpu(x.astype(np.float64) + 2.0 ** 30, dev), 3, 12)
        torch.cuda.synchronize()
        assert np.array_equal(a32.cpu().numpy(), a64.cpu().numpy())
        assert np.array_equal(a64.cpu().numpy(), orc.resample(scheme, x, 3, B=12)[1])


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("fusion", [True, False])
def test_f64_batched_paths(pf, dev, orc, scheme, fusion):
    """Batches through every dispatch of the float path, with ragged / odd row strides (the
    unvectorised loads), invalid filters (NaN, +inf, all -inf) and zero weights."""
    import torch

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    pf.pf_set_fusion(fusion)
    try:
        for N, P, ld in ((300, 200, 203), (40, 3000, 3000), (2 * sms, 8192, 8193), (3, 65536, 65536),
                         (1, (1 << 20) + 3, (1 << 20) + 4)):
            if scheme == "metropolis" and N * P > 3_000_000:
                continue
            x = pfinputs.gaussian_logw_f64(ld, 2.0, offset=-3.5e6, seed=N + P, N=N)
            x[:, ::17] = -np.inf
            x[:, 5::101] -= 1e300  # below float range after the shift: zero weight
            if N >= 3:
                x[0, P // 2] = np.nan
                x[N // 2, :] = -np.inf
                x[N - 1, P - 1] = np.inf
            g = _gpu(x, dev)[:, :P]
            st = torch.empty(N, dtype=torch.int32, device=dev)
            lse = torch.empty(N, dtype=torch.float64, device=dev)
            a = pf.pf_resample_batched(scheme, g, 99, B=10, first_filter=7, status_out=st, lse_out=lse)
            torch.cuda.synchronize()
            a, st, lse = a.cpu().numpy(), st.cpu().numpy(), lse.cpu().numpy()
            for n in range(N):
                wst, want, wlse, _, _ = orc.resample_f64(scheme, x[n, :P], 99, B=10, filter_index=7 + n, side=True)
                assert st[n] == wst, (N, P, n)
                assert np.array_equal(a[n], want), (scheme, N, P, n)
                if wst == 0:
                    assert abs(lse[n] - wlse) <= 1e-6
                else:
                    assert math.isnan(lse[n])
    finally:
        pf.pf_set_fusion(True)


@pytest.mark.parametrize("scheme", ["systematic", "stratified", "multinomial"])
def test_f64_permutation_and_state(pf, dev, orc, scheme):
    """offspring_out, permuted_out and the fused in-place state gather with binary64 weights
    (the pre-pass + cluster kernel at P = 4096, the binary64 cluster kernel itself at 8192 and
    65536 (gather fused / separate), the cooperative kernel's single large filter, the
    multi-launch path for multinomial)."""
    import torch

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    for N, P in ((2 * sms, 4096), (2 * sms, 8192), (5, 65536), (1, 300000)):
        x = pfinputs.gaussian_logw_f64(P, 1.0, offset=-1e7, seed=N, N=N)
        X = np.stack([pfinputs.state_matrix(P, 16, seed=n) for n in range(N)])
        gX = _gpu(X, dev)
        off = torch.empty((N, P), dtype=torch.int32, device=dev)
        perm = torch.empty((N, P), dtype=torch.int32, device=dev)
        a = pf.pf_resample_batched(scheme, _gpu(x, dev), 1234, first_filter=2, offspring_out=off, permuted_out=perm,
                                   state=gX)
        torch.cuda.synchronize()
        a, off, perm, gX = a.cpu().numpy(), off.cpu().numpy(), perm.cpu().numpy(), gX.cpu().numpy()
        for n in sorted({0, N // 2, N - 1}):
            _, want = orc.resample_f64(scheme, x[n], 1234, filter_index=2 + n)
            assert np.array_equal(a[n], want)
            assert np.array_equal(off[n], orc.ancestors_to_offspring(want))
            wp = orc.permute(want)
            assert np.array_equal(perm[n], wp)
            assert np.array_equal(gX[n], orc.gather_inplace(X[n], wp))


def test_f64_argument_errors(pf, dev):
    import torch

    lib = pf.lib()
    a = torch.empty(8, dtype=torch.int32, device=dev)
    x = torch.zeros(8, dtype=torch.float64, device=dev)
    n0 = pf.pf_launch_count()
    assert lib.pf_resample_ex_f64(3, None, 8, 1, 0, a.data_ptr(), None, None) == 1
    assert lib.pf_resample_ex_f64(3, x.data_ptr(), 0, 1, 0, a.data_ptr(), None, None) == 1
    assert lib.pf_resample_ex_f64(9, x.data_ptr(), 8, 1, 0, a.data_ptr(), None, None) == 1
    assert lib.pf_resample_batched_f64(3, x.data_ptr(), 4, 2, 8, 1, 0, 0, a.data_ptr(), 8, None,
                                       None) == 1
    assert pf.pf_launch_count() == n0


@pytest.mark.parametrize("scheme", ["systematic", "stratified", "multinomial"])
def test_f64_bench_size_sampled(pf, dev, orc, scheme):
    """The bench's binary64 extras at full C3 size (1024 filters x 2^16, offset -1e7, the
    binary64 cluster kernel for systematic / stratified, the pre-pass + bucket mode for
    multinomial): sampled filters against the oracle."""
    import torch

    N, P = 1024, 1 << 16
    x = pfinputs.gaussian_logw_torch(P, 1.0, 77, N, dev).double() - 1e7
    a = pf.pf_resample_batched(scheme, x, 2026, first_filter=5)
    torch.cuda.synchronize()
    for n in (0, 511, 1023):
        xn = x[n].cpu().numpy()
        assert np.array_equal(a[n].cpu().numpy(), orc.resample_f64(scheme, xn, 2026, filter_index=5 + n)[1]), n
