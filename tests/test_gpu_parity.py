"""GPU parity: the CUDA path (through the C-ABI binding) against the CPU oracle on the
same seeded inputs.  Bit-exact for ancestors / offspring / permutations / gathers;
lse, ess and normalised weights within 1e-6 relative (BJ north_star, NS-13).

Sizes span several 4096-particle tiles and ragged tails; the full BASELINE sizes
are checked in the launch configuration bench.py times (batched 1024 x 2^16) on
sampled filters, and single filters up to 2^24 in full.
"""
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


def _run(pf, dev, scheme, x, seed, B=0, filt=0, side=False, flags=0):
    import torch

    g = _gpu(x, dev)
    P = len(x)
    if flags and not side:
        a = pf.pf_resample_ex(scheme, g, seed, B, filter_index=filt, flags=flags)
        torch.cuda.synchronize()
        return a.cpu().numpy()
    if side:
        lse = torch.empty(1, dtype=torch.float64, device=dev)
        ess = torch.empty(1, dtype=torch.float64, device=dev)
        v = torch.empty(P, dtype=torch.float32, device=dev)
        st = torch.empty(1, dtype=torch.int32, device=dev)
        a = pf.pf_resample_ex(scheme, g, seed, B, filter_index=filt, lse_out=lse, ess_out=ess, normw_out=v,
                              status_out=st, flags=flags)
        torch.cuda.synchronize()
        return a.cpu().numpy(), float(lse.item()), float(ess.item()), v.cpu().numpy(), int(st.item())
    if filt == 0:
        fn = getattr(pf, f"pf_resample_{scheme}")
        a = fn(g, seed, B)
    else:
        a = pf.pf_resample_ex(scheme, g, seed, B, filter_index=filt)
    torch.cuda.synchronize()
    return a.cpu().numpy()


PS = [1, 2, 3, 7, 8, 16, 31, 1000, 4096, 4097, 12289, 65536, 100003]


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("var", [0.1, 1.0, 10.0])
def test_single_filter_bit_exact(pf, dev, orc, scheme, var):
    for P in PS:
        x = pfinputs.gaussian_logw(P, var, seed=P * 7 + int(var * 10))
        for seed in (1, pfinputs.seed_for(P)):
            B = 32 if scheme == "metropolis" else 0
            a = _run(pf, dev, scheme, x, seed, B)
            _, want = orc.resample(scheme, x, seed, B=B)
            assert np.array_equal(a, want), (scheme, var, P, seed, np.nonzero(a != want)[0][:5])


@pytest.mark.parametrize("scheme", ["stratified", "systematic"])
def test_multilaunch_path_bit_exact(pf, dev, orc, scheme):
    """The multi-launch path (k_max -> k_scan -> k_merge), forced with PF_NO_FUSION at sizes where the
    one-launch cluster kernel would otherwise run, is bit-exact too; side outputs included."""
    for P in (1, 2, 7, 16, 1000, 4097, 65536, 100003, 131072):
        for var in (0.1, 10.0):
            x = pfinputs.gaussian_logw(P, var, seed=P + 3)
            a = _run(pf, dev, scheme, x, 99, flags=pf.PF_NO_FUSION)
            _, want = orc.resample(scheme, x, 99)
            assert np.array_equal(a, want), (scheme, P, var)
            a, lse, ess, v, st = _run(pf, dev, scheme, x, 98, side=True, flags=pf.PF_NO_FUSION)
            _, want, wlse, wv, wess = orc.resample(scheme, x, 98, side=True)
            assert np.array_equal(a, want)
            assert abs(lse - wlse) <= 1e-6 * max(1.0, abs(wlse))


def test_multinomial_per_filter_scan(pf, dev, orc):
    """Batches that fill the GPU scan each filter in one CTA (no decoupled lookback): ragged sizes,
    -inf runs, heavy weights, an invalid filter; multinomial ancestors bit-exact against the oracle
    on sampled filters, lse within 1e-6."""
    import torch

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    for P, var in ((5000, 10.0), (4097, 1.0), (65536, 1.0), (100003, 0.1), (131072, 10.0), (300, 1.0)):
        N = sms + 3
        x = pfinputs.with_neg_inf_runs(pfinputs.gaussian_logw(P, var, seed=P, N=N))
        x[4, 11] = np.nan
        lse = torch.empty(N, dtype=torch.float64, device=dev)
        a = pf.pf_resample_batched("multinomial", _gpu(x, dev), 88, first_filter=2, lse_out=lse)
        torch.cuda.synchronize()
        A, L = a.cpu().numpy(), lse.cpu().numpy()
        for n in (0, 4, N // 2, N - 1):
            st, want, wl, _, _ = orc.resample("multinomial", x[n], 88, filter_index=2 + n, side=True)
            assert np.array_equal(A[n], want), (P, n)
            assert (st and np.isnan(L[n])) or abs(L[n] - wl) <= 1e-6 * max(1.0, abs(wl))


@pytest.mark.parametrize("scheme", ["stratified", "systematic"])
def test_large_filter_batches_dispatch(pf, dev, orc, scheme):
    """Filters above the cluster kernel's range: one filter takes the cooperative kernel (one
    launch), a batch of several takes the multi-launch path (the cooperative kernel serialises
    filters); both bit-exact against the oracle."""
    import torch

    P = 1 << 19
    x = pfinputs.gaussian_logw(P, 1.0, seed=77, N=3)
    g = _gpu(x, dev)
    c0 = pf.pf_launch_count()
    a1 = pf.pf_resample_batched(scheme, g[:1], 12, first_filter=40)
    torch.cuda.synchronize()
    assert pf.pf_launch_count() - c0 == 1
    c0 = pf.pf_launch_count()
    a3 = pf.pf_resample_batched(scheme, g, 12, first_filter=40)
    torch.cuda.synchronize()
    assert pf.pf_launch_count() - c0 > 1
    _, want = orc.resample_batched(scheme, x, 12, first_filter=40)
    assert np.array_equal(a3.cpu().numpy(), want)
    assert np.array_equal(a1.cpu().numpy(), want[:1])


@pytest.mark.parametrize("scheme", ["stratified", "systematic"])
def test_cluster_path_sizes(pf, dev, orc, scheme):
    """Cluster sizes 1..8 of the one-launch kernel (512 threads, P up to 8 x 8192) and 5..16 of its
    1024-thread form (P up to 16 x 16384, non-portable cluster sizes), ragged CTA ranges, skew."""
    import torch

    for P in (8191, 8192, 8193, 16384 + 5, 24576, 49152 + 3, 65535, 65536, 65537, 98304 + 7, 131072,
              131073, 200003, 262143, 262144):
        x = pfinputs.gaussian_logw(P, 10.0, seed=P)
        a = _run(pf, dev, scheme, x, 31)
        _, want = orc.resample(scheme, x, 31)
        assert np.array_equal(a, want), (scheme, P)
    # the 1024-thread form (clusters of 5..16) runs for batches that span the GPU
    for N, P in ((40, 65537), (20, 131072 + 5), (10, 262144)):
        x = pfinputs.gaussian_logw(P, 10.0, seed=P + N, N=N)
        c0 = pf.pf_launch_count()
        a = pf.pf_resample_batched(scheme, _gpu(x, dev), 32, first_filter=7)
        torch.cuda.synchronize()
        assert pf.pf_launch_count() - c0 == 1
        A = a.cpu().numpy()
        for n in (0, N // 2, N - 1):
            _, want = orc.resample(scheme, x[n], 32, filter_index=7 + n)
            assert np.array_equal(A[n], want), (scheme, N, P, n)
    # batched with more filters than resident clusters, ld > P, an invalid filter
    N, P, ld = 300, 20000, 20004
    x = pfinputs.gaussian_logw(ld, 1.0, seed=5, N=N)
    x[7, 100] = np.nan
    g = _gpu(x, dev)[:, :P]
    st = torch.empty(N, dtype=torch.int32, device=dev)
    lse = torch.empty(N, dtype=torch.float64, device=dev)
    a = pf.pf_resample_batched(scheme, g, 4, first_filter=1000, status_out=st, lse_out=lse)
    torch.cuda.synchronize()
    wst, want = orc.resample_batched(scheme, np.ascontiguousarray(x[:, :P]), 4, first_filter=1000)
    assert np.array_equal(st.cpu().numpy(), wst)
    assert np.array_equal(a.cpu().numpy(), want)
    for n in (0, 7, 299):
        _, _, wl, _, _ = orc.resample(scheme, np.ascontiguousarray(x[n, :P]), 4, filter_index=1000 + n, side=True)
        got = float(lse[n].item())
        assert (np.isnan(wl) and np.isnan(got)) or abs(got - wl) <= 1e-6 * max(1.0, abs(wl))


@pytest.mark.parametrize("scheme", SCHEMES)
def test_edge_cases_bit_exact(pf, dev, orc, scheme):
    cases = {
        "equal": pfinputs.equal_logw(4097, -2.0),
        "equal_pow2": pfinputs.equal_logw(8192, 5.0),
        "single_support": pfinputs.single_support_logw(9000, 8191),
        "single_support_first": pfinputs.single_support_logw(5000, 0),
        "single_support_last": pfinputs.single_support_logw(5000, 4999),
        "neg_inf_runs": pfinputs.with_neg_inf_runs(pfinputs.gaussian_logw(20000, 1.0, seed=5), frac=0.6),
        "huge_range": np.float32(pfinputs.gaussian_logw(10000, 1.0, seed=6) * 1e4),
        "subnormal_diffs": np.float32([1e-39, 0.0, -1e-39, 2e-39] * 100),
        "big_offset": pfinputs.gaussian_logw(3000, 1.0, seed=8) + np.float32(1e6),
        "dirichlet_0.01": pfinputs.dirichlet_logw(6000, 0.01, seed=3),
    }
    for name, x in cases.items():
        for B in ((0, 1, 7, 33) if scheme == "metropolis" else (0,)):
            a = _run(pf, dev, scheme, x, 12345, B)
            st, want = orc.resample(scheme, x, 12345, B=B)
            assert st == 0
            assert np.array_equal(a, want), (scheme, name, B)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_invalid_inputs(pf, dev, orc, scheme):
    for x in (np.float32([0, np.nan, 1, 2]), np.float32([0, np.inf] * 3000), np.full(5000, -np.inf, np.float32)):
        a, lse, ess, v, st = _run(pf, dev, scheme, x, 3, B=4, side=True)
        assert st == 1
        assert np.array_equal(a, np.arange(len(x)))
        assert math.isnan(lse) and math.isnan(ess) and np.all(np.isnan(v))


def test_argument_errors_enqueue_nothing(pf, dev):
    """include/pf.h error conventions: empty inputs (P = 0, N = 0), NULL pointers, B < 0, ld < P,
    a bad scheme and unknown flags are refused synchronously with the documented status and no
    kernel is enqueued."""
    import ctypes

    import torch

    L = pf.lib()
    x = torch.zeros(64, device=dev)
    a = torch.empty(64, dtype=torch.int32, device=dev)
    s0 = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    c0 = pf.pf_launch_count()
    INVALID, UNSUPPORTED = 1, 4
    assert L.pf_resample_systematic(x.data_ptr(), 0, 1, 0, a.data_ptr(), s0) == INVALID  # P = 0
    assert L.pf_resample_systematic(None, 64, 1, 0, a.data_ptr(), s0) == INVALID
    assert L.pf_resample_systematic(x.data_ptr(), 64, 1, 0, None, s0) == INVALID
    assert L.pf_resample_metropolis(x.data_ptr(), 64, 1, -1, a.data_ptr(), s0) == INVALID  # B < 0
    assert L.pf_resample_batched(3, x.data_ptr(), 8, 0, 8, 1, 0, 0, a.data_ptr(), 8, None, s0) == INVALID  # N = 0
    assert L.pf_resample_batched(3, x.data_ptr(), 7, 2, 8, 1, 0, 0, a.data_ptr(), 8, None, s0) == INVALID  # ld < P
    assert L.pf_resample_batched(3, x.data_ptr(), 8, 2, 8, 1, 0, 0, a.data_ptr(), 7, None, s0) == INVALID
    assert L.pf_resample_ex(9, x.data_ptr(), 64, 1, 0, a.data_ptr(), None, s0) == INVALID  # bad scheme
    opts = pf._Opts(flags=1 << 7)
    assert L.pf_resample_ex(3, x.data_ptr(), 64, 1, 0, a.data_ptr(), ctypes.byref(opts), s0) == UNSUPPORTED
    opts = pf._Opts(flags=pf.PF_SORTED)
    assert L.pf_resample_ex(3, x.data_ptr(), 64, 1, 0, a.data_ptr(), ctypes.byref(opts), s0) == UNSUPPORTED
    assert L.pf_ancestors_to_offspring(None, 64, a.data_ptr(), s0) == INVALID
    assert L.pf_permute(a.data_ptr(), 0, a.data_ptr(), s0) == INVALID
    assert pf.pf_launch_count() == c0
    assert pf.pf_status_string(INVALID) == "PF_ERR_INVALID_ARG"
    with pytest.raises(pf.PfError):
        pf.pf_resample_systematic(torch.zeros(0, device=dev), 1)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_side_outputs(pf, dev, orc, scheme):
    """lse, ess and normalised weights within 1e-6 relative of the oracle (NS-13)."""
    for P, var in ((1, 1.0), (16, 1.0), (4097, 10.0), (1 << 20, 1.0)):
        x = pfinputs.gaussian_logw(P, var, seed=P)
        a, lse, ess, v, st = _run(pf, dev, scheme, x, 9, B=8, side=True)
        _, want, wlse, wv, wess = orc.resample(scheme, x, 9, B=8, side=True)
        assert st == 0
        assert np.array_equal(a, want)
        assert abs(lse - wlse) <= 1e-6 * max(1.0, abs(wlse))
        assert abs(ess - wess) <= 1e-6 * wess
        assert np.all(np.abs(v - wv) <= 1e-6 * np.maximum(np.abs(wv), 1e-30))


def test_filter_index_streams(pf, dev, orc):
    x = pfinputs.gaussian_logw(5000, 1.0, seed=2)
    for scheme in SCHEMES:
        a = _run(pf, dev, scheme, x, 77, B=16, filt=123456)
        _, want = orc.resample(scheme, x, 77, B=16, filter_index=123456)
        assert np.array_equal(a, want)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_batched_bit_exact(pf, dev, orc, scheme):
    import torch

    for N, P, ld in ((3, 1, 1), (7, 1000, 1000), (5, 4097, 4100), (64, 4096, 4096), (9, 12289, 12300)):
        base = pfinputs.gaussian_logw(ld, 1.0, seed=N * P, N=N)
        x = pfinputs.with_neg_inf_runs(base)
        x[N // 2, :] = -np.inf  # one invalid filter in the batch
        g = _gpu(x, dev)[:, :P]
        st = torch.empty(N, dtype=torch.int32, device=dev)
        a = pf.pf_resample_batched(scheme, g, 4242, B=12, first_filter=17, status_out=st)
        torch.cuda.synchronize()
        a = a.cpu().numpy()
        wst, want = orc.resample_batched(scheme, np.ascontiguousarray(x[:, :P]), 4242, B=12, first_filter=17)
        assert np.array_equal(st.cpu().numpy(), wst)
        assert np.array_equal(a, want), (scheme, N, P)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_bench_config_sampled(pf, dev, orc, scheme):
    """BASELINE C3 at full size in the launch configuration bench.py times: 1024 filters x 2^16,
    sigma^2 = 1; sampled filters (incl. first and last) compared to the oracle in full."""
    import torch

    N, P = 1024, 1 << 16
    x = pfinputs.gaussian_logw_torch(P, 1.0, pfinputs.BASE_SEED, N, dev)
    B = 32 if scheme == "metropolis" else 0
    a = pf.pf_resample_batched(scheme, x, 0xC3, B=B, first_filter=0)
    torch.cuda.synchronize()
    for n in (0, 1, 511, 777, 1023):
        xn = x[n].cpu().numpy()
        _, want = orc.resample(scheme, xn, 0xC3, B=B, filter_index=n)
        assert np.array_equal(a[n].cpu().numpy(), want), (scheme, n)


@pytest.mark.parametrize("scheme", ["systematic", "stratified"])
def test_bench_step_sampled(pf, dev, orc, scheme):
    """The exact step bench.py times (C3 at full size: 1024 filters x 2^16, sigma^2 = 1, one
    pf_resample_batched call with offspring, permutation and the D = 16 state gather, one launch);
    sampled filters checked in full against the oracle: ancestors, offspring, permutation, rows."""
    import torch

    N, P, D = 1024, 1 << 16, 16
    x = pfinputs.gaussian_logw_torch(P, 1.0, pfinputs.BASE_SEED, N, dev)
    X = torch.randn((N, P, D), generator=torch.Generator(device=dev).manual_seed(1), device=dev)
    X0 = {n: X[n].cpu().numpy() for n in (0, 3, 500, 1023)}
    anc = torch.empty((N, P), dtype=torch.int32, device=dev)
    off = torch.empty_like(anc)
    perm = torch.empty_like(anc)
    c0 = pf.pf_launch_count()
    pf.pf_resample_batched(scheme, x, pfinputs.seed_for(0), ancestors=anc, offspring_out=off, permuted_out=perm,
                           state=X)
    torch.cuda.synchronize()
    assert pf.pf_launch_count() - c0 == 1
    for n, Xn in X0.items():
        _, want = orc.resample(scheme, x[n].cpu().numpy(), pfinputs.seed_for(0), filter_index=n)
        assert np.array_equal(anc[n].cpu().numpy(), want), n
        assert np.array_equal(off[n].cpu().numpy(), orc.ancestors_to_offspring(want)), n
        wp = orc.permute(want)
        assert np.array_equal(perm[n].cpu().numpy(), wp), n
        assert np.array_equal(X[n].cpu().numpy(), orc.gather_inplace(Xn, wp)), n
    del X


def test_host_pipeline_matches_direct_call(pf, dev, orc):
    """paper_1202_6163_b200.pipeline.HostPipeline (chunked, overlapped H2D / kernel / D2H on three
    streams) returns exactly what one direct call does, for several chunk counts and schemes,
    including the device state gathered in place; checked against the oracle for sampled filters."""
    import torch

    from paper_1202_6163_b200.pipeline import HostPipeline

    N, P, D = 37, 3000, 16
    x = pfinputs.gaussian_logw(P, 1.0, seed=21, N=N)
    h_logw = torch.from_numpy(x).pin_memory()
    X0 = torch.randn((N, P, D), generator=torch.Generator().manual_seed(3))
    for scheme in ("systematic", "multinomial"):
        Xd = _gpu(X0.numpy(), dev)
        ref_perm = torch.empty((N, P), dtype=torch.int32, device=dev)
        pf.pf_resample_batched(scheme, _gpu(x, dev), 77, first_filter=5, permuted_out=ref_perm, state=Xd)
        torch.cuda.synchronize()
        for chunks in (1, 3, 8):
            pipe = HostPipeline(N, P, dev, chunks=chunks)
            Xp = _gpu(X0.numpy(), dev)
            h_out = torch.empty((N, P), dtype=torch.int32).pin_memory()
            pipe.run(scheme, h_logw, 77, h_out, first_filter=5, state=Xp)
            torch.cuda.synchronize()
            assert torch.equal(h_out, ref_perm.cpu()), (scheme, chunks)
            assert torch.equal(Xp, Xd), (scheme, chunks)
            # chained calls (the next batch's input copies overlap this one's output copies):
            # two different batches back to back, each equal to its own direct call
            h2 = torch.from_numpy(pfinputs.gaussian_logw(P, 10.0, seed=22, N=N)).pin_memory()
            ref2 = torch.empty((N, P), dtype=torch.int32, device=dev)
            pf.pf_resample_batched(scheme, h2.to(dev), 78, first_filter=5, permuted_out=ref2)
            o1 = torch.empty((N, P), dtype=torch.int32).pin_memory()
            o2 = torch.empty((N, P), dtype=torch.int32).pin_memory()
            for _ in range(2):
                pipe.run(scheme, h_logw, 77, o1, first_filter=5, chain=True)
                pipe.run(scheme, h2, 78, o2, first_filter=5, chain=True)
            torch.cuda.synchronize()
            assert torch.equal(o1, ref_perm.cpu()) and torch.equal(o2, ref2.cpu()), (scheme, chunks)
        for n in (0, 36):
            _, want = orc.resample(scheme, x[n], 77, filter_index=5 + n)
            assert np.array_equal(ref_perm[n].cpu().numpy(), orc.permute(want))


@pytest.mark.parametrize("scheme", ["systematic", "stratified", "multinomial", "sorted", "metropolis"])
def test_maximum_sizes(pf, dev, orc, scheme):
    """Maximum sizes: a batch of 2^15 filters x 2^16 = 2^31 particles (8 GiB of log-weights; 64-bit
    indexing of rows, tiles and workspace) with sampled filters checked in full, and a single filter
    of 2^28 + 3 particles with sampled slots (chains) checked against the oracle."""
    import torch

    sch = "multinomial" if scheme == "sorted" else scheme
    flags = pf.PF_SORTED if scheme == "sorted" else 0
    B = 4 if scheme == "metropolis" else 0
    N, P = 1 << 15, 1 << 16
    x = pfinputs.gaussian_logw_torch(P, 1.0, 99, N, dev)
    a = pf.pf_resample_batched(sch, x, 0x5EED, B=B, first_filter=3, flags=flags)
    torch.cuda.synchronize()
    for n in (0, 1, N // 2 + 1, N - 1):
        xn = x[n].cpu().numpy()
        if scheme == "sorted":
            _, want = orc.resample_sorted_multinomial(xn, 0x5EED, filter_index=3 + n)
        else:
            _, want = orc.resample(sch, xn, 0x5EED, B=B, filter_index=3 + n)
        assert np.array_equal(a[n].cpu().numpy(), want), (scheme, n)
    del x, a
    torch.cuda.empty_cache()
    if scheme == "sorted":
        return  # the oracle's 2^28-spacings scan would dominate the test; the batch above covers a6
    P1 = (1 << 28) + 3
    g = pfinputs.gaussian_logw_torch(P1, 1.0, 7, 1, dev)[0].contiguous()
    a = pf.pf_resample_ex(sch, g, 0xB16, B, filter_index=1)
    torch.cuda.synchronize()
    xh = g.cpu().numpy()
    rng = np.random.default_rng(1)
    ks = np.unique(np.concatenate([[0, 1, P1 - 2, P1 - 1], rng.integers(0, P1, 2000)]))
    ah = a[torch.from_numpy(ks).to(dev)].cpu().numpy()
    if scheme == "metropolis":
        _, w = orc.weights(xh)
        for k, got in zip(ks[:300], ah[:300]):
            assert got == orc.metropolis_chains(w, int(k), 1, 0xB16, B, 1)[0], int(k)
        return
    _, Q = orc.cumulative(xh)
    Qtot = int(Q[-1])
    for k, got in zip(ks, ah):
        want = orc.upper_bound(Q, orc.position(sch, P1, Qtot, 0xB16, 1, int(k)))
        assert got == want, (scheme, int(k))
    if scheme != "multinomial":
        assert bool((a[1:] >= a[:-1]).all())


@pytest.mark.parametrize("P", [1 << 20, (1 << 22) + 12345, 1 << 24])
def test_large_single_filter(pf, dev, orc, P):
    """C2 (2^20) and larger single filters in full, all prefix-sum schemes; Metropolis on sampled chains."""
    import torch

    x = pfinputs.gaussian_logw(P, 10.0 if P > (1 << 22) else 1.0, seed=P)
    g = _gpu(x, dev)
    for scheme in ("multinomial", "stratified", "systematic"):
        a = getattr(pf, f"pf_resample_{scheme}")(g, 555).cpu().numpy()
        _, want = orc.resample(scheme, x, 555)
        assert np.array_equal(a, want), scheme
    a = pf.pf_resample_metropolis(g, 556, 32).cpu().numpy()
    st, w = orc.weights(x)
    rng = np.random.default_rng(0)
    idx = np.unique(np.concatenate([[0, P - 1], rng.integers(0, P, 3000)]))
    for i in idx:
        assert a[i] == orc.metropolis_chains(w, int(i), 1, 556, 32)[0]


def test_offspring_permute_gather(pf, dev, orc):
    import torch

    rng = np.random.default_rng(1)
    for P in (1, 2, 5, 1000, 4097, 65536, 100003):
        for scheme in ("multinomial", "systematic", "metropolis"):
            x = pfinputs.gaussian_logw(P, float(rng.choice([0.1, 1.0, 10.0])), seed=P)
            _, anc = orc.resample(scheme, x, 5, B=3)
            anc = rng.permutation(anc).astype(np.int32) if scheme == "multinomial" else anc
            ga = _gpu(anc, dev)
            o = pf.pf_ancestors_to_offspring(ga)
            perm = pf.pf_permute(ga)
            torch.cuda.synchronize()
            assert np.array_equal(o.cpu().numpy(), orc.ancestors_to_offspring(anc))
            want_perm = orc.permute(anc)
            assert np.array_equal(perm.cpu().numpy(), want_perm), (P, scheme)
            for D in (16, 3):
                X = pfinputs.state_matrix(P, D, seed=P)
                gX = _gpu(X, dev)
                pf.pf_gather_state(gX, perm)
                Y = pf.pf_gather_state_out(_gpu(X, dev), ga)
                torch.cuda.synchronize()
                assert np.array_equal(gX.cpu().numpy(), orc.gather_inplace(X, want_perm))
                assert np.array_equal(Y.cpu().numpy(), orc.gather_out(X, anc))


@pytest.mark.parametrize("fusion", [True, False])
def test_permute_paths(pf, dev, orc, fusion):
    """Both permutation paths (cluster kernel, and the multi-launch hist -> lookback scan -> merge path
    forced with pf_set_fusion(False)) against the oracle: sorted and unsorted ancestors, heavy
    particles (sigma^2 = 10), ragged sizes, batched with ld > P."""
    import torch

    pf.pf_set_fusion(fusion)
    try:
        rng = np.random.default_rng(2)
        for P in (1, 3, 8, 4096, 8191, 8193, 30000, 65536):
            for scheme, var in (("systematic", 10.0), ("multinomial", 1.0), ("stratified", 0.1)):
                x = pfinputs.gaussian_logw(P, var, seed=P + 1)
                _, anc = orc.resample(scheme, x, 17)
                if scheme == "multinomial":
                    anc = rng.permutation(anc).astype(np.int32)
                perm = pf.pf_permute(_gpu(anc, dev))
                torch.cuda.synchronize()
                assert np.array_equal(perm.cpu().numpy(), orc.permute(anc)), (fusion, P, scheme)
        N, P, ld = 21, 12000, 12004
        x = pfinputs.gaussian_logw(P, 1.0, seed=4, N=N)
        _, A = orc.resample_batched("systematic", x, 5)
        Ag = torch.zeros((N, ld), dtype=torch.int32, device=dev)
        Ag[:, :P] = _gpu(A, dev)
        out = torch.full((N, ld), -7, dtype=torch.int32, device=dev)
        pf.pf_permute(Ag[:, :P], permuted=out[:, :P])
        torch.cuda.synchronize()
        o = out.cpu().numpy()
        for n in range(N):
            assert np.array_equal(o[n, :P], orc.permute(A[n]))
        assert np.all(o[:, P:] == -7)
    finally:
        pf.pf_set_fusion(True)


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("fusion", [True, False])
def test_offspring_out_and_permute_offspring(pf, dev, orc, scheme, fusion):
    """pf_opts.offspring_out (fused: derived from slot counts; otherwise the histogram) equals the
    oracle's offspring, and pf_permute_offspring equals the oracle's canonical permutation."""
    import torch

    pf.pf_set_fusion(fusion)
    try:
        for N, P, var in ((1, 1, 1.0), (1, 7, 1.0), (3, 4097, 10.0), (16, 65536, 1.0), (2, 100003, 0.1)):
            x = pfinputs.gaussian_logw(P, var, seed=P, N=N)
            if N > 2:
                x[1, :] = -np.inf  # an invalid filter: identity ancestors, offspring 1
            g = _gpu(x, dev)
            off = torch.empty((N, P), dtype=torch.int32, device=dev)
            B = 9 if scheme == "metropolis" else 0
            a = pf.pf_resample_batched(scheme, g, 71, B=B, offspring_out=off)
            perm = pf.pf_permute_offspring(off)
            torch.cuda.synchronize()
            _, want = orc.resample_batched(scheme, x, 71, B=B)
            assert np.array_equal(a.cpu().numpy(), want)
            O = off.cpu().numpy()
            Pm = perm.cpu().numpy()
            for n in range(N):
                assert np.array_equal(O[n], orc.ancestors_to_offspring(want[n])), (scheme, N, P, n)
                assert np.array_equal(Pm[n], orc.permute(want[n])), (scheme, N, P, n)
    finally:
        pf.pf_set_fusion(True)


def test_offspring_histogram_batches(pf, dev, orc):
    """The shared-memory histogram (two CTAs per filter, batches of >= half the SMs, P <= 65536):
    offspring of random, skewed (one particle takes every slot) and identity ancestors, odd P,
    ld > P, against the oracle; and the permutation built on it."""
    import torch

    rng = np.random.default_rng(7)
    for N, P in ((200, 65536), (150, 5001), (100, 2), (90, 777)):
        ld = P + 4
        A = rng.integers(0, P, size=(N, ld)).astype(np.int32)
        A[1, :P] = P - 1            # every slot on the last particle (count = P)
        A[2, :P] = np.arange(P)     # identity
        A[3, :P] = 0                # every slot on particle 0
        g = _gpu(A, dev)[:, :P]
        o = pf.pf_ancestors_to_offspring(g)
        pm = pf.pf_permute(g)
        torch.cuda.synchronize()
        O, Pm = o.cpu().numpy(), pm.cpu().numpy()
        for n in (0, 1, 2, 3, N - 1):
            assert np.array_equal(O[n], orc.ancestors_to_offspring(A[n, :P])), (N, P, n)
            assert np.array_equal(Pm[n], orc.permute(A[n, :P])), (N, P, n)


def test_batched_offspring_permute_gather(pf, dev, orc):
    import torch

    N, P, D = 33, 5000, 16
    x = pfinputs.gaussian_logw(P, 1.0, seed=1, N=N)
    _, A = orc.resample_batched("multinomial", x, 8)
    gA = _gpu(A, dev)
    O = pf.pf_ancestors_to_offspring(gA)
    Pm = pf.pf_permute(gA)
    X = np.stack([pfinputs.state_matrix(P, D, seed=n) for n in range(N)])
    gX = _gpu(X, dev)
    pf.pf_gather_state(gX, Pm)
    torch.cuda.synchronize()
    for n in range(N):
        assert np.array_equal(O[n].cpu().numpy(), orc.ancestors_to_offspring(A[n]))
        wp = orc.permute(A[n])
        assert np.array_equal(Pm[n].cpu().numpy(), wp)
        assert np.array_equal(gX[n].cpu().numpy(), orc.gather_inplace(X[n], wp))


@pytest.mark.parametrize("scheme", SCHEMES)
def test_fused_state_gather(pf, dev, orc, scheme):
    """pf_opts.state: the in-place state gather with the canonical permutation (NS-15/16), fused
    into the cluster kernel (power-of-two rows of 16..512 bytes) or run after the permutation
    (other schemes / sizes / row layouts).  Rows, ancestors, offspring and permutation bit-exact
    against the oracle; padding between rows and filters untouched; an invalid filter."""
    import torch

    B = 5 if scheme == "metropolis" else 0
    cases = [(3, 1000, 16, 16), (5, 8192, 4, 4), (2, 8193, 16, 20), (4, 65536, 128, 128), (2, 30000, 3, 3),
             (1, 100003, 16, 16), (3, 200, 8, 8), (1, 1, 16, 16), (2, 1 << 18, 16, 16), (1, 300000, 16, 16),
             (150, 3000, 16, 16), (20, 65536, 16, 16), (10, 1 << 18, 16, 16)]
    for N, P, D, ldD in cases:
        x = pfinputs.gaussian_logw(P, 1.0, seed=P + D, N=N)
        if N > 2:
            x[1, 7] = np.nan
        X = np.stack([np.pad(pfinputs.state_matrix(P, D, seed=n), ((0, 0), (0, ldD - D)), constant_values=-3.0)
                      for n in range(N)])
        Xp = np.concatenate([X, np.full((N, 5, ldD), -9.0, np.float32)], axis=1)  # filter padding rows
        gXp = _gpu(Xp, dev)
        gX = gXp[:, :P, :D]
        off = torch.empty((N, P), dtype=torch.int32, device=dev)
        perm = torch.empty((N, P), dtype=torch.int32, device=dev)
        c0 = pf.pf_launch_count()
        a = pf.pf_resample_batched(scheme, _gpu(x, dev), 29, B=B, offspring_out=off, permuted_out=perm, state=gX)
        torch.cuda.synchronize()
        nl = pf.pf_launch_count() - c0
        cl = -(-P // 8192) if P <= 65536 else -(-P // 16384)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        if scheme in ("stratified", "systematic") and (P <= 65536 or (P <= (1 << 18) and N * cl >= sms)):
            # one cluster-kernel launch; the gather is fused when the batch spans the GPU (N x cluster
            # CTAs >= SMs) and the rows allow it, else it follows as one more launch
            fused = D * 4 in (16, 32, 64, 128, 256, 512) and D == ldD and N * cl >= sms
            assert nl == (1 if fused else 2), (N, P, D, nl)
        _, want = orc.resample_batched(scheme, x, 29, B=B)
        assert np.array_equal(a.cpu().numpy(), want)
        got = gXp.cpu().numpy()
        for n in range(N):
            wp = orc.permute(want[n])
            assert np.array_equal(perm[n].cpu().numpy(), wp)
            assert np.array_equal(off[n].cpu().numpy(), orc.ancestors_to_offspring(want[n]))
            assert np.array_equal(got[n, :P, :D], orc.gather_inplace(X[n, :, :D], wp)), (scheme, N, P, D, n)
        assert np.all(got[:, :P, D:] == -3.0) and np.all(got[:, P:] == -9.0)
    # state without permuted_out / offspring_out (fused path writes neither)
    N, P, D = 4, 20000, 16
    x = pfinputs.gaussian_logw(P, 10.0, seed=3, N=N)
    X = np.stack([pfinputs.state_matrix(P, D, seed=n + 50) for n in range(N)])
    gX = _gpu(X, dev)
    a = pf.pf_resample_batched(scheme, _gpu(x, dev), 30, B=B, state=gX)
    torch.cuda.synchronize()
    _, want = orc.resample_batched(scheme, x, 30, B=B)
    assert np.array_equal(a.cpu().numpy(), want)
    for n in range(N):
        assert np.array_equal(gX[n].cpu().numpy(), orc.gather_inplace(X[n], orc.permute(want[n])))


@pytest.mark.parametrize("scheme", SCHEMES + ["sorted"])
def test_explicit_workspace(pf, dev, orc, scheme):
    """pf_opts.workspace: a caller buffer of pf_workspace_bytes(_ex) bytes serves every path the
    dispatch takes (warp / CTA / cluster / cooperative / multi-launch kernels; the permutation
    scratch of the fused state gather); results equal the pool's; too small or misaligned buffers
    and the unsupported combination (permutation on the multi-launch path) are refused."""
    import torch

    sch = "multinomial" if scheme == "sorted" else scheme
    flags = pf.PF_SORTED if scheme == "sorted" else 0
    B = 7 if scheme == "metropolis" else 0
    for N, P in ((300, 16), (3, 700), (5, 6000), (2, 65536), (1, 300000), (4, 300000)):
        x = pfinputs.gaussian_logw(P, 1.0, seed=N + P, N=N)
        g = _gpu(x, dev)
        nbytes = pf.pf_workspace_bytes(sch, N, P, flags=flags)
        assert nbytes > 0
        ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=dev)
        off = (-ws.data_ptr()) % 256
        wsv = ws[off:off + nbytes]
        a = pf.pf_resample_batched(sch, g, 41, B=B, flags=flags, workspace=wsv)
        torch.cuda.synchronize()
        _, want = orc.resample_batched(sch, x, 41, B=B) if scheme != "sorted" else (None, np.stack(
            [orc.resample_sorted_multinomial(x[n], 41, filter_index=n)[1] for n in range(N)]))
        assert np.array_equal(a.cpu().numpy(), want), (scheme, N, P)
        if scheme in ("stratified", "systematic") and P <= 65536:
            X = torch.randn((N, P, 16), device=dev)
            X0 = X.cpu().numpy()
            pf.pf_resample_batched(sch, g, 41, state=X, workspace=wsv)
            torch.cuda.synchronize()
            for n in range(N):
                assert np.array_equal(X[n].cpu().numpy(), orc.gather_inplace(X0[n], orc.permute(want[n])))
    # refusals
    x = _gpu(pfinputs.gaussian_logw(5000, 1.0, seed=1, N=2), dev)
    tiny = torch.empty(256, dtype=torch.uint8, device=dev)
    need_ws = scheme in ("multinomial", "sorted", "metropolis")
    if need_ws:
        with pytest.raises(pf.PfError):
            pf.pf_resample_batched(sch, _gpu(pfinputs.gaussian_logw(300000, 1.0, seed=2, N=2), dev), 1, B=B,
                                   flags=flags, workspace=tiny)
    big = torch.empty(pf.pf_workspace_bytes(sch, 2, 300000, flags=flags) + 512, dtype=torch.uint8, device=dev)
    mis = big[((-big.data_ptr()) % 256) + 8:]
    with pytest.raises(pf.PfError):
        pf.pf_resample_batched(sch, _gpu(pfinputs.gaussian_logw(300000, 1.0, seed=2, N=2), dev), 1, B=B, flags=flags,
                               workspace=mis)
    if need_ws:
        perm = torch.empty((2, 5000), dtype=torch.int32, device=dev)
        with pytest.raises(pf.PfError):
            pf.pf_resample_batched(sch, x, 1, B=B, flags=flags, permuted_out=perm, workspace=big)


def test_repeatability_and_launch_count(pf, dev):
    import torch

    x = _gpu(pfinputs.gaussian_logw(1 << 16, 1.0, seed=3), dev)
    c0 = pf.pf_launch_count()
    a1 = pf.pf_resample_stratified(x, 11).clone()
    a2 = pf.pf_resample_stratified(x, 11)
    torch.cuda.synchronize()
    assert torch.equal(a1, a2)
    assert pf.pf_launch_count() - c0 == 2  # one cluster kernel per call (P <= 8 x 8192)
    c0 = pf.pf_launch_count()
    pf.pf_resample_ex("stratified", x, 11, flags=pf.PF_NO_FUSION)
    torch.cuda.synchronize()
    assert pf.pf_launch_count() - c0 == 3  # max, scan, merge


@pytest.mark.parametrize("scheme", SCHEMES)
def test_giant_filter_fake_shards(pf, dev, orc, scheme):
    """C5 decomposition on one GPU (fake-shard mode): the shard kernels (pf_shard_max / scan / search,
    pf_shard_weights, pf_metropolis_from_weights) with host-side exchanges reproduce the single-filter
    result bit-exactly, for several shard counts, a shard without weight, and an invalid filter."""
    import torch

    from paper_1202_6163_b200.shard import resample_sharded_local, shard_range

    B = 16 if scheme == "metropolis" else 0
    cases = [(1000, 2, 1.0, ""), (4097, 3, 10.0, ""), (65536, 8, 1.0, ""), (100003, 5, 0.1, ""),
             (1 << 20, 8, 1.0, ""), (9000, 4, 1.0, "neg_inf_shard"), (5000, 2, 1.0, "invalid")]
    for P, G, var, kind in cases:
        x = pfinputs.gaussian_logw(P, var, seed=P + G)
        if kind == "neg_inf_shard":
            p0, Pl = shard_range(P, G, 2)
            x[p0:p0 + Pl] = -np.inf
        if kind == "invalid":
            x[17] = np.inf
        g = _gpu(x, dev)
        a = resample_sharded_local(scheme, g, G, 4321, B=B, filter_index=3)
        torch.cuda.synchronize()
        _, want = orc.resample(scheme, x, 4321, B=B, filter_index=3)
        assert np.array_equal(a.cpu().numpy(), want), (scheme, P, G, kind)


def test_giant_filter_fake_shards_sorted_multinomial(pf, dev, orc):
    """C5 decomposition of the sorted multinomial (a6) on one GPU: spacing totals per
    spacing shard, device-side plan, range scan of the spacings, merge.  Bit-exact against the
    oracle's single-filter run for several shard counts, weight-skewed shards (one shard holding
    almost all weight, so its slot range spans many spacing shards), a shard without weight and
    an invalid filter."""
    import torch

    from paper_1202_6163_b200.shard import PF_SORTED, resample_sharded_local, shard_range

    cases = [(1000, 2, 1.0, ""), (4097, 3, 10.0, ""), (65536, 8, 1.0, ""), (100003, 5, 0.1, ""),
             (1 << 20, 8, 1.0, ""), (9000, 4, 1.0, "neg_inf_shard"), (5000, 2, 1.0, "invalid"),
             (200000, 8, 1.0, "skew"), (7, 3, 1.0, ""), (1, 1, 1.0, ""), (3, 2, 1.0, "")]
    for P, G, var, kind in cases:
        x = pfinputs.gaussian_logw(P, var, seed=P + G + 1)
        if kind == "neg_inf_shard":
            p0, Pl = shard_range(P, G, 2)
            x[p0:p0 + Pl] = -np.inf
        if kind == "invalid":
            x[17] = np.inf
        if kind == "skew":
            p0, Pl = shard_range(P, G, 5)
            x[p0:p0 + Pl] += 12.0  # shard 5 holds nearly all the weight
        g = _gpu(x, dev)
        a = resample_sharded_local("multinomial", g, G, 1234, filter_index=4, flags=PF_SORTED)
        torch.cuda.synchronize()
        _, want = orc.resample_sorted_multinomial(x, 1234, filter_index=4)
        assert np.array_equal(a.cpu().numpy(), want), (P, G, kind)


MIGRATION_SCHEMES = [("systematic", 0), ("stratified", 0), ("multinomial", 0), ("multinomial", 1), ("metropolis", 0)]


@pytest.mark.parametrize("scheme,flags", MIGRATION_SCHEMES)
def test_particle_migration_ranks_on_one_gpu(pf, dev, orc, scheme, flags):
    """Cross-GPU particle migration (include/pf.h 4a-4d; NEXT-4): G ranks run as threads on one
    GPU through the real resample_sharded(assemble=False) + migrate_sharded code (slot ranges,
    Metropolis reduce-scatter of slot histograms, split sizes, all-to-all by slicing).  Every
    rank's rows and permutation slice equal the oracle's whole-filter permute + in-place gather,
    element by element; a shard without weight (all its slots refilled from other shards), a
    weight-skewed shard and an invalid filter (nothing moves) included."""
    import torch

    from paper_1202_6163_b200.shard import GpuStages, migrate_sharded, resample_sharded, shard_range
    from tests._loopback_comm import run_ranks

    B = 16 if scheme == "metropolis" else 0
    cases = [(1000, 2, 1.0, ""), (4097, 3, 10.0, ""), (100003, 5, 1.0, ""), (1 << 18, 8, 1.0, ""),
             (9000, 4, 1.0, "neg_inf_shard"), (20000, 4, 1.0, "skew"), (5000, 2, 1.0, "invalid"), (7, 3, 1.0, "")]
    for P, G, var, kind in cases:
        x = pfinputs.gaussian_logw(P, var, seed=P + G + 7)
        if kind == "neg_inf_shard":
            p0, Pl = shard_range(P, G, 1)
            x[p0:p0 + Pl] = -np.inf
        if kind == "skew":
            p0, Pl = shard_range(P, G, 2)
            x[p0:p0 + Pl] += 8.0
        if kind == "invalid":
            x[3] = np.nan
        X = pfinputs.state_matrix(P, 16, seed=P)

        def rank_fn(r, comm):
            p0, Pl = shard_range(P, G, r)
            anc, info = resample_sharded(scheme, _gpu(x[p0:p0 + Pl], dev), P, 777, B=B, filter_index=9, comm=comm,
                                         stages=GpuStages(), assemble=False, flags=flags)
            Xl = _gpu(X[p0:p0 + Pl], dev)
            perm = migrate_sharded(Xl, anc, info, comm=comm)
            return Xl.cpu().numpy(), perm.cpu().numpy()

        out = run_ranks(G, rank_fn)
        if flags:
            _, want = orc.resample_sorted_multinomial(x, 777, filter_index=9)
        else:
            _, want = orc.resample(scheme, x, 777, B=B, filter_index=9)
        wp = orc.permute(want)
        assert np.array_equal(np.concatenate([p for _, p in out]), wp), (scheme, P, G, kind)
        assert np.array_equal(np.concatenate([a for a, _ in out]), orc.gather_inplace(X, wp)), (scheme, P, G, kind)


def test_particle_migration_layouts(pf, dev, orc):
    """Migration stages on fake shards (migrate_sharded_local) for every copy width: 64-byte
    float rows (16-byte chunks), 12-byte rows (4-byte chunks), 7-byte rows (bytes), rows with a
    stride wider than the row, indices only; ancestors from the oracle with extreme offspring
    (one particle takes every slot; the identity); P = 2^20 over 8 shards; argument errors."""
    import torch

    from paper_1202_6163_b200.shard import migrate_sharded_local

    def check(Xh, anc, G, X_dev=None):
        wp = orc.permute(anc)
        Xd = X_dev if X_dev is not None else (_gpu(Xh, dev) if Xh is not None else None)
        perm = migrate_sharded_local(Xd, _gpu(anc, dev), G)
        torch.cuda.synchronize()
        assert np.array_equal(perm.cpu().numpy(), wp), (G, len(anc))
        if Xh is not None:
            got = Xd.cpu().numpy()
            assert np.array_equal(got, orc.gather_inplace(Xh, wp)), (G, len(anc), Xh.dtype, Xh.shape)

    P = 5003
    x = pfinputs.gaussian_logw(P, 1.0, seed=5)
    _, anc = orc.resample("stratified", x, 31)
    check(pfinputs.state_matrix(P, 16), anc, 3)
    check(pfinputs.state_matrix(P, 3), anc, 4)
    rng = np.random.default_rng(1)
    check(rng.integers(0, 255, size=(P, 7), dtype=np.uint8), anc, 2)
    check(None, anc, 5)
    wide = pfinputs.state_matrix(P, 20)
    Xw = _gpu(wide, dev)
    wp = orc.permute(anc)
    perm = migrate_sharded_local(Xw[:, :16], _gpu(anc, dev), 3)
    torch.cuda.synchronize()
    want = wide.copy()
    want[:, :16] = orc.gather_inplace(np.ascontiguousarray(wide[:, :16]), wp)
    assert np.array_equal(Xw.cpu().numpy(), want)
    check(pfinputs.state_matrix(P, 16), np.full(P, P - 2, dtype=np.int32), 4)  # one particle takes all
    # one particle takes every slot of a 2^20 filter: its shard's 2^20 - 1 extras are split into
    # work items over many CTAs (the pack side was one CTA per tile)
    Pd = 1 << 20
    check(pfinputs.state_matrix(Pd, 16), np.full(Pd, 3, dtype=np.int32), 8)
    check(pfinputs.state_matrix(P, 16), np.arange(P, dtype=np.int32), 4)  # nothing moves
    Pb = 1 << 20
    _, ancb = orc.resample("systematic", pfinputs.gaussian_logw(Pb, 1.0, seed=8), 3)
    check(pfinputs.state_matrix(Pb, 16), ancb, 8)
    a = _gpu(anc, dev)
    o = torch.empty(P, dtype=torch.int32, device=dev)
    L = pf.lib()
    assert L.pf_shard_offspring(a.data_ptr(), P, None, 0, 0, None, None, o.data_ptr(), None) == 1
    assert L.pf_shard_offspring(a.data_ptr(), P, None, 0, P, None, a.data_ptr(), o.data_ptr(), None) == 1
    plan = torch.empty(L.pf_shard_migration_plan_bytes(P) // 8, dtype=torch.int64, device=dev)
    assert L.pf_shard_migration_counts(o.data_ptr(), 0, plan.data_ptr(), o.data_ptr(), None) == 1
    assert L.pf_shard_migration_counts(o.data_ptr(), P, None, o.data_ptr(), None) == 1
    assert L.pf_shard_migrate_pack(None, 64, 64, P, 0, o.data_ptr(), plan.data_ptr(), None, None, None) == 1
    assert L.pf_shard_migrate_pack(None, 0, 0, P, 0, o.data_ptr(), None, None, a.data_ptr(), None) == 1
    assert L.pf_shard_migrate_unpack(None, 0, 0, P, 0, o.data_ptr(), plan.data_ptr(), None, a.data_ptr(), None,
                                     None) == 1
    assert L.pf_shard_migrate_unpack(None, 64, 64, P, 0, o.data_ptr(), plan.data_ptr(), None, None, None, None) == 1


def test_sorted_multinomial_a6(pf, dev, orc):
    """a6 (PF_SORTED with the multinomial): spacings scan + exact 128/64 positions + merge,
    bit-exact against the oracle; batched with ld > P and an invalid filter; ragged sizes."""
    import torch

    for P in (1, 2, 3, 7, 16, 1000, 4095, 4096, 4097, 65536, 100003, 1 << 20):
        for var in ((1.0, 10.0) if P < (1 << 20) else (1.0,)):
            x = pfinputs.with_neg_inf_runs(pfinputs.gaussian_logw(P, var, seed=P + 9))
            a = pf.pf_resample_ex("multinomial", _gpu(x, dev), 2718, filter_index=6, flags=pf.PF_SORTED)
            torch.cuda.synchronize()
            _, want = orc.resample_sorted_multinomial(x, 2718, filter_index=6)
            assert np.array_equal(a.cpu().numpy(), want), (P, var)
    N, P, ld = 9, 5000, 5003
    x = pfinputs.gaussian_logw(ld, 1.0, seed=2, N=N)
    x[4, 10] = np.nan
    g = _gpu(x, dev)[:, :P]
    st = torch.empty(N, dtype=torch.int32, device=dev)
    A = pf.pf_resample_batched("multinomial", g, 31, first_filter=100, flags=pf.PF_SORTED, status_out=st)
    torch.cuda.synchronize()
    A = A.cpu().numpy()
    for n in range(N):
        s_, want = orc.resample_sorted_multinomial(np.ascontiguousarray(x[n, :P]), 31, filter_index=100 + n)
        assert int(st[n].item()) == s_
        assert np.array_equal(A[n], want), n


@pytest.mark.parametrize("scheme", SCHEMES + ["sorted"])
def test_small_filters_warp_kernel(pf, dev, orc, scheme):
    """P <= 256: the one-warp-per-filter kernel (every scheme, a6 included) against the oracle,
    batched with invalid filters, ld > P, side outputs and offspring; and the same cases through the
    multi-launch path (pf_set_fusion(False))."""
    import torch

    for fusion in (True, False):
        pf.pf_set_fusion(fusion)
        try:
            for N, P in ((1, 16), (1000, 16), (333, 100), (64, 256), (7, 1), (50, 33)):
                ld = P + 3
                x = pfinputs.gaussian_logw(ld, 1.0 if N % 2 else 10.0, seed=N * P, N=N)
                if N > 10:
                    x[5, 0] = np.nan
                    x[6, :] = -np.inf
                g = _gpu(x, dev)[:, :P]
                st = torch.empty(N, dtype=torch.int32, device=dev)
                lse = torch.empty(N, dtype=torch.float64, device=dev)
                off = torch.empty((N, P), dtype=torch.int32, device=dev)
                sch = "multinomial" if scheme == "sorted" else scheme
                flags = pf.PF_SORTED if scheme == "sorted" else 0
                B = 21 if scheme == "metropolis" else 0
                a = pf.pf_resample_batched(sch, g, 99, B=B, first_filter=3, status_out=st, lse_out=lse,
                                           offspring_out=off, flags=flags)
                torch.cuda.synchronize()
                A, O, S, L = a.cpu().numpy(), off.cpu().numpy(), st.cpu().numpy(), lse.cpu().numpy()
                for n in range(N):
                    xn = np.ascontiguousarray(x[n, :P])
                    if scheme == "sorted":
                        s_, want = orc.resample_sorted_multinomial(xn, 99, filter_index=3 + n)
                        wl = L[n] if s_ else orc.resample("systematic", xn, 1, side=True)[2]
                    else:
                        s_, want, wl, _, _ = orc.resample(sch, xn, 99, B=B, filter_index=3 + n, side=True)
                    assert S[n] == s_ and np.array_equal(A[n], want), (fusion, scheme, N, P, n)
                    assert np.array_equal(O[n], orc.ancestors_to_offspring(want))
                    assert (np.isnan(wl) and np.isnan(L[n])) or abs(L[n] - wl) <= 1e-6 * max(1.0, abs(wl))
        finally:
            pf.pf_set_fusion(True)


@pytest.mark.parametrize("scheme", SCHEMES + ["sorted"])
def test_medium_filters_cta_kernel(pf, dev, orc, scheme):
    """256 < P <= 8192: the one-CTA-per-filter kernel (every scheme, a6 included; one launch; taken
    up to P = 1024 always, above per the measured dispatch rule) and whatever the dispatch picks
    above it, against the oracle: ragged sizes, batched with invalid filters, ld > P, -inf runs,
    heavy weights, side outputs (lse, ESS, normalised weights, status) and offspring."""
    import torch

    sch = "multinomial" if scheme == "sorted" else scheme
    flags = pf.PF_SORTED if scheme == "sorted" else 0
    B = 13 if scheme == "metropolis" else 0
    for N, P in ((1, 257), (1, 1000), (3, 4096), (2, 4097), (5, 8191), (1, 8192), (40, 777)):
        ld = P + 5
        x = pfinputs.with_neg_inf_runs(pfinputs.gaussian_logw(ld, 1.0 if N % 2 else 10.0, seed=N + P, N=N))
        if N > 4:
            x[2, 9] = np.nan
            x[3, :] = -np.inf
        g = _gpu(x, dev)[:, :P]
        st = torch.empty(N, dtype=torch.int32, device=dev)
        lse = torch.empty(N, dtype=torch.float64, device=dev)
        ess = torch.empty(N, dtype=torch.float64, device=dev)
        nw = torch.empty((N, P), dtype=torch.float32, device=dev)
        off = torch.empty((N, P), dtype=torch.int32, device=dev)
        c0 = pf.pf_launch_count()
        a = pf.pf_resample_batched(sch, g, 1234, B=B, first_filter=9, status_out=st, lse_out=lse, ess_out=ess,
                                   normw_out=nw, offspring_out=off, flags=flags)
        torch.cuda.synchronize()
        if P <= 1024:
            assert pf.pf_launch_count() - c0 == 1, (scheme, N, P)
        A, O, S, L, E, V = (a.cpu().numpy(), off.cpu().numpy(), st.cpu().numpy(), lse.cpu().numpy(),
                            ess.cpu().numpy(), nw.cpu().numpy())
        for n in range(N):
            xn = np.ascontiguousarray(x[n, :P])
            s_, w_, wl, wv, we = orc.resample("systematic", xn, 1, side=True)
            if scheme == "sorted":
                s_, want = orc.resample_sorted_multinomial(xn, 1234, filter_index=9 + n)
            else:
                s_, want = orc.resample(sch, xn, 1234, B=B, filter_index=9 + n)
            assert S[n] == s_ and np.array_equal(A[n], want), (scheme, N, P, n)
            assert np.array_equal(O[n], orc.ancestors_to_offspring(want))
            if s_:
                assert np.isnan(L[n]) and np.isnan(E[n])
                continue
            assert abs(L[n] - wl) <= 1e-6 * max(1.0, abs(wl))
            assert abs(E[n] - we) <= 1e-6 * we
            assert np.all(np.abs(V[n] - wv) <= 1e-6 * np.maximum(np.abs(wv), 1e-30) + 1e-12)


def test_lg_step_layouts_agree(pf, dev):
    """The C4 propagate + weight kernel gives identical states and log-weights on 16-byte-aligned
    rows (float4 path) and on unaligned rows (scalar path)."""
    import torch

    P, D = 5000, 16
    Xa = torch.empty((P, D), device=dev)
    pf.pf_lg_init(Xa, 0.9, 1.0, 77)
    Xb = torch.zeros((P, D + 1), device=dev)[:, :D]  # ld = 17 floats: not 16-byte aligned rows
    Xb.copy_(Xa)
    for t in (1, 2, 3):
        la = pf.pf_lg_propagate_weight(Xa, 0.9, 1.0, 1.0, 0.3 * t, 77, t)
        lb = pf.pf_lg_propagate_weight(Xb, 0.9, 1.0, 1.0, 0.3 * t, 77, t)
        torch.cuda.synchronize()
        assert torch.equal(la, lb) and torch.equal(Xa, Xb), t


def test_pf_linear_gaussian_c4(pf, dev, orc):
    """C4: bootstrap PF (propagate + weight kernels, resample, permute, gather) on the 16-dim
    linear-Gaussian model: log-likelihood within Monte Carlo error of the Kalman filter, and every
    checked step's resampling bit-exact against the oracle fed the GPU's log-weights."""
    from oracle.kalman import kalman_loglik
    from paper_1202_6163_b200.pf_demo import LinearGaussianPF

    T = 40
    ys = pfinputs.lg_observations(T, seed=5)
    want, _ = kalman_loglik(ys)
    lls = [LinearGaussianPF(P=1 << 16, seed=100 + r).run(ys) for r in range(6)]
    mean, sd = float(np.mean(lls)), float(np.std(lls, ddof=1))
    assert abs(mean - want) < 5 * sd / math.sqrt(len(lls)) + 0.05, (mean, want, sd)
    for scheme in ("systematic", "stratified", "multinomial", "metropolis"):
        f = LinearGaussianPF(P=5000, seed=9, scheme=scheme, B=16 if scheme == "metropolis" else 0)
        for y in ys[:4]:
            logw, anc, s = f.step(float(y), check=True)
            _, wanted = orc.resample(scheme, logw, s, B=f.B)
            assert np.array_equal(anc, wanted), scheme


@pytest.mark.parametrize("scheme", SCHEMES + ["sorted"])
def test_permuted_out(pf, dev, orc, scheme):
    """pf_opts.permuted_out (fused into the cluster kernel for stratified/systematic, P <= 65536;
    resample + permutation from offspring otherwise) equals the oracle's canonical permutation of the
    oracle's ancestors; batched, ragged, with an invalid filter; with and without offspring_out."""
    import torch

    sch = "multinomial" if scheme == "sorted" else scheme
    flags = pf.PF_SORTED if scheme == "sorted" else 0
    B = 13 if scheme == "metropolis" else 0
    for N, P, var in ((1, 100, 1.0), (5, 8192, 10.0), (3, 8193, 1.0), (12, 30000, 1.0), (2, 65536, 10.0),
                      (1, 100003, 1.0)):
        ld = P + 4
        x = pfinputs.gaussian_logw(ld, var, seed=N + P, N=N)
        if N > 3:
            x[2, :] = -np.inf
        g = _gpu(x, dev)[:, :P]
        for with_off in (False, True):
            perm = torch.full((N, ld), -5, dtype=torch.int32, device=dev)[:, :P]
            off = torch.empty((N, ld), dtype=torch.int32, device=dev)[:, :P] if with_off else None
            anc = torch.empty((N, ld), dtype=torch.int32, device=dev)[:, :P]
            pf.pf_resample_batched(sch, g, 8, B=B, first_filter=2, ancestors=anc, offspring_out=off,
                                   permuted_out=perm, flags=flags)
            torch.cuda.synchronize()
            A, Pm = anc.cpu().numpy(), perm.cpu().numpy()
            for n in range(N):
                xn = np.ascontiguousarray(x[n, :P])
                if scheme == "sorted":
                    _, want = orc.resample_sorted_multinomial(xn, 8, filter_index=2 + n)
                else:
                    _, want = orc.resample(sch, xn, 8, B=B, filter_index=2 + n)
                assert np.array_equal(A[n], want), (scheme, N, P, n)
                assert np.array_equal(Pm[n], orc.permute(want)), (scheme, N, P, n, with_off)
                if with_off:
                    assert np.array_equal(off.cpu().numpy()[n], orc.ancestors_to_offspring(want))


def _heavy_logw(P, seed):
    """Skewed log-weights with runs that cover whole expansion chunks: particle 0 holds 1/32 of
    the mass (its ~P/32 slots and extras ranks start at 0, a chunk boundary), particles 7, 8 and
    P/2 (one sub-tile / another CTA) 1/16, 1/64 and 1/8 each, the rest sigma^2 = 1 far below."""
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal(P) - 12.0).astype(np.float32)
    rest = float(np.sum(np.exp(x.astype(np.float64))))
    heavy = {0: 1 / 32, 7: 1 / 16, 8: 1 / 64, P // 2: 1 / 8}
    light = 1.0 - sum(heavy.values())
    for i, f in heavy.items():
        x[i] = np.float32(np.log(f / light * rest))
    return x


@pytest.mark.parametrize("P", [1 << 18, (1 << 20) + 3])
def test_heavy_runs_cooperative_kernel(pf, dev, orc, P):
    """Slot-balanced expansion (the cooperative kernel's deferred runs, kinds slots and extras
    ranks): ancestors, offspring and the canonical permutation of filters whose heavy particles'
    runs cover whole chunks, including one that starts at a chunk boundary, bit-exact vs the
    oracle; plus the sigma^2 = 10 filter of C2."""
    import torch

    for x in (_heavy_logw(P, 3), pfinputs.gaussian_logw(P, 10.0, seed=P + 1)):
        g = _gpu(x, dev)
        for scheme in ("systematic", "stratified"):
            off = torch.empty(P, dtype=torch.int32, device=dev)
            pm = torch.empty(P, dtype=torch.int32, device=dev)
            a = pf.pf_resample_ex(scheme, g, 77, offspring_out=off, permuted_out=pm)
            torch.cuda.synchronize()
            _, want = orc.resample(scheme, x, 77)
            assert np.array_equal(a.cpu().numpy(), want), (scheme, P)
            assert np.array_equal(off.cpu().numpy(), orc.ancestors_to_offspring(want)), (scheme, P)
            assert np.array_equal(pm.cpu().numpy(), orc.permute(want)), (scheme, P)
        # batched form (several filters through the same deferred lists, both parities)
        xb = np.stack([x, x[::-1].copy(), x])
        ab = pf.pf_resample_batched("systematic", _gpu(xb, dev), 5)
        torch.cuda.synchronize()
        for n in range(3):
            _, want = orc.resample("systematic", xb[n], 5, filter_index=n)
            assert np.array_equal(ab[n].cpu().numpy(), want), n


@pytest.mark.parametrize("N,P", [(24, 1 << 16), (160, 4099), (40, 40001)])
def test_fused_permutation_from_offspring(pf, dev, orc, N, P):
    """a9 + a10 from offspring counts in one cluster-kernel launch (the multinomial / Metropolis
    step, pf_permute_batched, pf_permute_offspring_batched) for batches that span the GPU:
    permutations and gathered states bit-exact vs the oracle, incl. ragged P and an invalid
    filter (identity)."""
    import torch

    xb = pfinputs.gaussian_logw(P, 1.0, seed=N + P, N=N)
    xb[1, 5] = np.nan  # NS-1: this filter's ancestors, offspring and permutation are the identity
    X = np.stack([pfinputs.state_matrix(P, 16, seed=n) for n in range(N)])
    for scheme, B in (("multinomial", 0), ("metropolis", 9)):
        gX = _gpu(X, dev)
        off = torch.empty((N, P), dtype=torch.int32, device=dev)
        pm = torch.empty((N, P), dtype=torch.int32, device=dev)
        n0 = pf.pf_launch_count()
        a = pf.pf_resample_batched(scheme, _gpu(xb, dev), 41, B=B, offspring_out=off, permuted_out=pm, state=gX)
        torch.cuda.synchronize()
        _, want = orc.resample_batched(scheme, xb, 41, B=B)
        assert np.array_equal(a.cpu().numpy(), want), scheme
        pmh, Xh = pm.cpu().numpy(), gX.cpu().numpy()
        for n in range(N):
            wp = orc.permute(want[n])
            assert np.array_equal(pmh[n], wp), (scheme, n)
            assert np.array_equal(Xh[n], orc.gather_inplace(X[n], wp)), (scheme, n)
        assert pf.pf_launch_count() > n0
        # the standalone conversions take the same kernel
        p2 = pf.pf_permute(_gpu(want, dev))
        p3 = pf.pf_permute_offspring(_gpu(np.stack([orc.ancestors_to_offspring(want[n]) for n in range(N)]), dev))
        torch.cuda.synchronize()
        for n in (0, 1, N - 1):
            wp = orc.permute(want[n])
            assert np.array_equal(p2[n].cpu().numpy(), wp) and np.array_equal(p3[n].cpu().numpy(), wp), (scheme, n)


def test_routed_multinomial_matches_replicated(pf, dev, orc):
    """The routed multinomial stages (pf_shard_route_count / pack / search) and the replicated
    pf_shard_search give the same ancestors, shard by shard (fake shards), and the oracle's."""
    import torch

    from paper_1202_6163_b200.shard import GpuStages, resample_sharded_local, shard_range

    st = GpuStages()
    for P, G in ((20011, 4), (1 << 18, 8)):
        x = pfinputs.gaussian_logw(P, 1.0, seed=P)
        g = _gpu(x, dev)
        routed = resample_sharded_local("multinomial", g, G, 99, filter_index=2)
        parts = [shard_range(P, G, h) for h in range(G)]
        mx = [st.max(g[p0:p0 + Pl]) for p0, Pl in parts]
        gmax = torch.stack([m for m, _ in mx]).max(dim=0).values
        gbad = torch.stack([b for _, b in mx]).max(dim=0).values
        scans = [st.scan(g[p0:p0 + Pl], P, gmax) for p0, Pl in parts]
        totals = torch.cat([t for _, t, _ in scans])
        rep = torch.full((P,), -1, dtype=torch.int32, device=dev)
        for h, ((p0, _), (Q, _, _)) in enumerate(zip(parts, scans)):
            st.search(1, Q, p0, P, totals, h, gmax, gbad, 99, 2, rep)
        torch.cuda.synchronize()
        _, want = orc.resample("multinomial", x, 99, filter_index=2)
        assert np.array_equal(routed.cpu().numpy(), want), (P, G)
        assert np.array_equal(rep.cpu().numpy(), want), (P, G)


@pytest.mark.parametrize("D", [16, 3, 6])
def test_lg_step_elementwise(pf, dev, orc, D):
    """C4 propagate + weight kernel (k_lg_step, k_lg_init) element by element against the
    oracle/lg_model.py step from the same input state (NS-18): states within 1e-5 (1 + |x|),
    log-weights within 1e-5 (1 + |logw|) of the binary64 oracle (the kernel's binary32 arithmetic
    and <= 2-ulp library functions), for the float4 rows (D = 16) and the scalar rows."""
    import torch

    from oracle import lg_model

    P, phi, sx, sy, seed = 3001, 0.9, 1.0, 1.0, 0x5EED
    X = torch.empty((P, D), device=dev)
    pf.pf_lg_init(X, phi, sx, seed)
    torch.cuda.synchronize()
    X0 = lg_model.lg_init(P, D, phi, sx, seed)
    assert np.allclose(X.cpu().numpy(), X0, rtol=0, atol=1e-5 * (1 + np.abs(X0).max()))
    for t, y in ((0, 0.3), (17, -2.5)):
        Xin = X.cpu().numpy().astype(np.float64)
        logw = pf.pf_lg_propagate_weight(X, phi, sx, sy, y, seed, t)
        torch.cuda.synchronize()
        Xw, lw = lg_model.lg_step(Xin, y, t, phi, sx, sy, seed)
        got = X.cpu().numpy()
        assert np.all(np.abs(got - Xw) <= 1e-5 * (1 + np.abs(Xw))), (D, t)
        assert np.all(np.abs(logw.cpu().numpy() - lw) <= 1e-5 * (1 + np.abs(lw))), (D, t)
