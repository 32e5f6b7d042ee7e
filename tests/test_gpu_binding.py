"""The binding is the only place that sees tensor sizes (the C ABI takes raw pointers): every
caller buffer a call writes is checked for dtype, device, layout and size before the call, and
an undersized one raises PfError with nothing enqueued."""
from __future__ import annotations

import pytest

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


def test_undersized_buffers_raise(pf):
    import torch

    dev = torch.device("cuda:0")
    P, N = 1000, 4
    x = torch.randn(P, device=dev)
    xb = torch.randn(N, P, device=dev)
    small = torch.empty(P - 1, dtype=torch.int32, device=dev)
    n0 = pf.pf_launch_count()
    for kw in ({"ancestors": small}, {"offspring_out": small}, {"permuted_out": small},
               {"normw_out": torch.empty(P - 1, device=dev)},
               {"state": torch.zeros(P - 1, 16, device=dev)}):
        with pytest.raises(pf.PfError):
            pf.pf_resample_ex("systematic", x, 1, **kw)
    with pytest.raises(pf.PfError):
        pf.pf_resample_systematic(x, 1, ancestors=small)
    a_small = torch.empty(N, P - 1, dtype=torch.int32, device=dev)
    a_rows = torch.empty(N - 1, P, dtype=torch.int32, device=dev)
    for kw in ({"ancestors": a_small}, {"ancestors": a_rows}, {"offspring_out": a_rows},
               {"permuted_out": a_small},
               {"lse_out": torch.empty(N - 1, dtype=torch.float64, device=dev)},
               {"status_out": torch.empty(N - 1, dtype=torch.int32, device=dev)},
               {"normw_out": torch.empty(N * P - 1, device=dev)},
               {"state": torch.zeros(N, P - 1, 16, device=dev)},
               # offspring / permutation rows are written with the ancestors' row stride
               {"offspring_out": torch.empty(N, P + 4, dtype=torch.int32, device=dev)[:, :P]}):
        with pytest.raises(pf.PfError):
            pf.pf_resample_batched("systematic", xb, 1, **kw)
    anc = torch.zeros(P, dtype=torch.int32, device=dev)
    with pytest.raises(pf.PfError):
        pf.pf_ancestors_to_offspring(anc, small)
    with pytest.raises(pf.PfError):
        pf.pf_permute(anc, small)
    with pytest.raises(pf.PfError):
        pf.pf_permute_offspring(anc, small)
    with pytest.raises(pf.PfError):
        pf.pf_gather_state(torch.zeros(P - 1, 16, device=dev), anc)
    with pytest.raises(pf.PfError):
        pf.pf_gather_state_out(torch.zeros(P, 16, device=dev), anc, torch.zeros(P - 1, 16, device=dev))
    ab = torch.zeros(N, P, dtype=torch.int32, device=dev)
    with pytest.raises(pf.PfError):
        pf.pf_ancestors_to_offspring(ab, a_small)
    with pytest.raises(pf.PfError):
        pf.pf_gather_state(torch.zeros(N, P - 1, 4, device=dev), ab)
    torch.cuda.synchronize()
    assert pf.pf_launch_count() == n0  # nothing was enqueued


def test_right_sized_views_still_work(pf):
    """Wider rows (ld > P) with matching strides are accepted (the checks are not too strict)."""
    import torch

    dev = torch.device("cuda:0")
    N, P = 3, 777
    xb = torch.randn(N, P + 5, device=dev)[:, :P]
    a = torch.full((N, P + 9), -1, dtype=torch.int32, device=dev)[:, :P]
    o = torch.full((N, P + 9), -1, dtype=torch.int32, device=dev)[:, :P]
    pf.pf_resample_batched("stratified", xb, 3, ancestors=a, offspring_out=o)
    torch.cuda.synchronize()
    assert int(o.sum()) == N * P
