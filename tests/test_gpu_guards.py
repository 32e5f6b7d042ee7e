"""Out-of-bounds write guards for the paths added late in round 1 (compute-sanitizer is not
available on the GPU pool): every output row has a sentinel-filled tail (ld > P) and every
flat output a sentinel-filled margin; after the call the sentinels must be untouched and the
in-bounds values must equal the oracle's."""
from __future__ import annotations

import numpy as np
import pytest

import pfinputs

pytestmark = pytest.mark.gpu
SENT = -77


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


CASES = [
    # (label, scheme, flags, N, P, input dtype)
    ("f64 cluster", "systematic", 0, 30, 12289, "f64"),
    ("f64 cluster", "stratified", 0, 3, 65536, "f64"),
    ("f64 prepass", "metropolis", 0, 5, 3001, "f64"),
    ("sorted weights one tile", "stratified", "sortw", 9, 4096, "f32"),
    ("sorted weights tiles", "multinomial", "sortw", 3, 20001, "f32"),
    ("bucket cluster", "multinomial", 0, 20, 12289, "f32"),
    ("bucket cluster", "multinomial", 0, 1, 4097, "f32"),
    ("bucket coop", "multinomial", 0, 1, 70001, "f32"),
]


@pytest.mark.parametrize("label,scheme,flags,N,P,dt", CASES)
def test_no_writes_out_of_bounds(pf, dev, orc, label, scheme, flags, N, P, dt):
    import torch

    ld = P + 37
    if dt == "f64":
        x = pfinputs.gaussian_logw_f64(P, 1.0, offset=-1e6, seed=P, N=N)
    else:
        x = pfinputs.gaussian_logw(P, 2.0, seed=P, N=N)
    fl = pf.PF_SORT_WEIGHTS if flags == "sortw" else 0
    anc_buf = torch.full((N, ld), SENT, dtype=torch.int32, device=dev)
    off_buf = torch.full((N, ld), SENT, dtype=torch.int32, device=dev)
    nw_flat = torch.full((N * P + 64,), float(SENT), dtype=torch.float32, device=dev)
    st_flat = torch.full((N + 16,), SENT, dtype=torch.int32, device=dev)
    lse_flat = torch.full((N + 16,), float(SENT), dtype=torch.float64, device=dev)
    use_normw = scheme != "metropolis"
    pf.pf_resample_batched(scheme, torch.from_numpy(x).to(dev), 11, B=6, first_filter=2, ancestors=anc_buf[:, :P],
                           offspring_out=off_buf[:, :P], status_out=st_flat[:N], lse_out=lse_flat[:N],
                           normw_out=nw_flat[:N * P].view(N, P) if use_normw else None, flags=fl)
    torch.cuda.synchronize()
    a = anc_buf.cpu().numpy()
    o = off_buf.cpu().numpy()
    assert np.all(a[:, P:] == SENT) and np.all(o[:, P:] == SENT), label
    assert np.all(nw_flat[N * P:].cpu().numpy() == SENT)
    assert np.all(st_flat[N:].cpu().numpy() == SENT) and np.all(lse_flat[N:].cpu().numpy() == SENT)
    for n in sorted({0, N - 1}):
        if dt == "f64":
            want = orc.resample_f64(scheme, x[n], 11, B=6, filter_index=2 + n)[1]
        elif fl:
            want = orc.resample_sorted_weights(scheme, x[n], 11, filter_index=2 + n)[1]
        else:
            want = orc.resample(scheme, x[n], 11, B=6, filter_index=2 + n)[1]
        assert np.array_equal(a[n, :P], want), (label, n)
        assert np.array_equal(o[n, :P], orc.ancestors_to_offspring(want))
