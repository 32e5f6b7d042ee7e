"""paper_1202_6163_b200 — Python binding of libpfresample (include/pf.h).

Argument marshalling only: every step of the resampling path runs in the
sm_100a kernels of ``libpfresample.so``.  There is NO CPU fallback: if the
library or a CUDA device is missing, every entry point raises.

Function names are the C names (``pf_resample_systematic``...).  Tensors are
torch CUDA tensors (PyTorch supplies device memory and streams only); the
stream defaults to torch's current stream on the tensor's device.

Citations: P:n = PAPER.md line n; NS-n = DESIGN.md §3.
"""
from __future__ import annotations

import ctypes
import os

from ._build import LIB as _LIB_PATH

# diagnostics only (tools/variants.py A/B builds): another build of the same library
_LIB_PATH = os.environ.get("PF_LIB_OVERRIDE", _LIB_PATH)

PF_MULTINOMIAL, PF_STRATIFIED, PF_SYSTEMATIC, PF_METROPOLIS = 1, 2, 3, 4
SCHEMES = {"multinomial": 1, "stratified": 2, "systematic": 3, "metropolis": 4}
PF_FILTER_OK, PF_FILTER_INVALID_WEIGHTS = 0, 1
PF_SORTED = 1 << 0  # pf_opts.flags with multinomial: sorted-uniform variant (a6, NS-12)
PF_NO_FUSION = 1 << 1  # pf_opts.flags: force the multi-launch path (diagnostics)
PF_SORT_WEIGHTS = 1 << 2  # pf_opts.flags: the paper's pre-sorted weight series (NS-17)


class PfError(RuntimeError):
    pass


class _Opts(ctypes.Structure):
    _fields_ = [
        ("filter_index", ctypes.c_uint32),
        ("flags", ctypes.c_uint32),
        ("lse_out", ctypes.c_void_p),
        ("normw_out", ctypes.c_void_p),
        ("ess_out", ctypes.c_void_p),
        ("status_out", ctypes.c_void_p),
        ("offspring_out", ctypes.c_void_p),
        ("permuted_out", ctypes.c_void_p),
        ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_size_t),
        ("state", ctypes.c_void_p),
        ("state_row_bytes", ctypes.c_int64),
        ("state_ld_bytes", ctypes.c_int64),
        ("state_filter_ld_bytes", ctypes.c_int64),
    ]


_lib = None

# (name, argtypes, restype) of every exported symbol of include/pf.h
_V, _I32, _U32, _I64, _U64, _F64, _SZ = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_int64,
                                         ctypes.c_uint64, ctypes.c_double, ctypes.c_size_t)
_SIGS = {
    "pf_resample_multinomial": ([_V, _I32, _U64, _I32, _V, _V], ctypes.c_int),
    "pf_resample_stratified": ([_V, _I32, _U64, _I32, _V, _V], ctypes.c_int),
    "pf_resample_systematic": ([_V, _I32, _U64, _I32, _V, _V], ctypes.c_int),
    "pf_resample_metropolis": ([_V, _I32, _U64, _I32, _V, _V], ctypes.c_int),
    "pf_resample_ex": ([ctypes.c_int, _V, _I32, _U64, _I32, _V, _V, _V], ctypes.c_int),
    "pf_resample_batched": ([ctypes.c_int, _V, _I64, _I32, _I32, _U64, _U32, _I32, _V, _I64, _V, _V], ctypes.c_int),
    "pf_resample_ex_f64": ([ctypes.c_int, _V, _I32, _U64, _I32, _V, _V, _V], ctypes.c_int),
    "pf_resample_batched_f64": ([ctypes.c_int, _V, _I64, _I32, _I32, _U64, _U32, _I32, _V, _I64, _V, _V],
                                ctypes.c_int),
    "pf_workspace_bytes": ([ctypes.c_int, _I32, _I32], _SZ),
    "pf_workspace_bytes_ex": ([ctypes.c_int, _I32, _I32, _U32, _I64], _SZ),
    "pf_ancestors_to_offspring": ([_V, _I32, _V, _V], ctypes.c_int),
    "pf_ancestors_to_offspring_batched": ([_V, _I64, _I32, _I32, _V, _I64, _V], ctypes.c_int),
    "pf_permute": ([_V, _I32, _V, _V], ctypes.c_int),
    "pf_permute_batched": ([_V, _I64, _I32, _I32, _V, _I64, _V], ctypes.c_int),
    "pf_permute_offspring": ([_V, _I32, _V, _V], ctypes.c_int),
    "pf_permute_offspring_batched": ([_V, _I64, _I32, _I32, _V, _I64, _V], ctypes.c_int),
    "pf_gather_state": ([_V, _I64, _I64, _I32, _V, _V], ctypes.c_int),
    "pf_gather_state_batched": ([_V, _I64, _I64, _I64, _I32, _I32, _V, _I64, _V], ctypes.c_int),
    "pf_gather_state_out": ([_V, _V, _I64, _I64, _I64, _I32, _V, _V], ctypes.c_int),
    "pf_shard_max": ([_V, _I32, _V, _V, _V], ctypes.c_int),
    "pf_shard_scan": ([_V, _I32, _I64, _V, _V, _V, _V, _V], ctypes.c_int),
    "pf_shard_route_count": ([_V, _I32, _I32, _I64, _V, _V, _U64, _U32, _V, _V], ctypes.c_int),
    "pf_shard_route_pack": ([_V, _I32, _I32, _I64, _V, _V, _U64, _U32, _V, _V, _V, _V], ctypes.c_int),
    "pf_shard_route_search": ([_V, _I32, _I64, _I64, _V, _I32, _I32, _V, _V, _V, _V, _I64, _V, _V], ctypes.c_int),
    "pf_shard_search": ([ctypes.c_int, _V, _I32, _I64, _I64, _V, _I32, _I32, _V, _V, _U64, _U32, _V, _V, _V],
                        ctypes.c_int),
    "pf_shard_spacings_total": ([_I64, _I32, _I32, _U64, _U32, _V, _V], ctypes.c_int),
    "pf_shard_search_sorted_workspace_bytes": ([_I64], _SZ),
    "pf_shard_search_sorted": ([_V, _I32, _I64, _I64, _V, _V, _I32, _I32, _V, _V, _U64, _U32, _V, _V, _V, _SZ, _V],
                               ctypes.c_int),
    "pf_shard_weights": ([_V, _I32, _V, _V, _V], ctypes.c_int),
    "pf_metropolis_from_weights": ([_V, _I64, _I64, _I32, _U64, _I32, _U32, _V, _V, _V, _V], ctypes.c_int),
    "pf_shard_offspring": ([_V, _I64, _V, _I64, _I32, _V, _V, _V, _V], ctypes.c_int),
    "pf_shard_migration_plan_bytes": ([_I32], _SZ),
    "pf_shard_migration_counts": ([_V, _I32, _V, _V, _V], ctypes.c_int),
    "pf_shard_migrate_pack": ([_V, _I64, _I64, _I32, _I64, _V, _V, _V, _V, _V], ctypes.c_int),
    "pf_shard_migrate_unpack": ([_V, _I64, _I64, _I32, _I64, _V, _V, _V, _V, _V, _V], ctypes.c_int),
    "pf_lg_init": ([_V, _I64, _I32, _I32, ctypes.c_float, ctypes.c_float, _U64, _V], ctypes.c_int),
    "pf_lg_propagate_weight": ([_V, _I64, _I32, _I32, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                ctypes.c_float, _U64, _I32, _V, _V], ctypes.c_int),
    "pf_lg_accumulate": ([_V, _I32, ctypes.c_float, _V, _V], ctypes.c_int),
    "pf_metropolis_required_B": ([_I64, _F64, _F64], _I32),
    "pf_status_string": ([ctypes.c_int], ctypes.c_char_p),
    "pf_launch_count": ([], _U64),
    "pf_profile_enable": ([_I32], None),
    "pf_set_fusion": ([_I32], None),
    "pf_profile_collect": ([_V, _I32], _I32),
    "pf_version": ([], ctypes.c_char_p),
    "pf_release": ([], None),
}


def library_path() -> str:
    return _LIB_PATH


def lib():
    """Load libpfresample.so (built in-tree by __graft_entry__.build()).  Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise PfError(f"libpfresample.so not built at {_LIB_PATH}: run __graft_entry__.build() "
                          "(there is no CPU fallback)")
        L = ctypes.CDLL(_LIB_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def _check(rc: int, what: str):
    if rc != 0:
        msg = lib().pf_status_string(rc).decode()
        raise PfError(f"{what} failed: {msg}")


def _torch():
    import torch

    return torch


def _stream(t, stream):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream(t.device)
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _need_cuda(t, dtype, name):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise PfError(f"{name} must be a CUDA tensor (libpfresample has no CPU path)")
    if t.dtype != dtype:
        raise PfError(f"{name} must be {dtype}, got {t.dtype}")


def _same_device(t, ref, name):
    if t.device != ref.device:
        raise PfError(f"{name} is on {t.device}, logw on {ref.device}: every buffer of a call must be on one device")


def _need_vec(t, dtype, name, ref, n):
    """A caller buffer the library writes n elements of, densely: right dtype, same device as
    logw, contiguous, at least n elements (the C ABI cannot see tensor sizes)."""
    _need_cuda(t, dtype, name)
    _same_device(t, ref, name)
    if not t.is_contiguous():
        raise PfError(f"{name} must be contiguous")
    if t.numel() < n:
        raise PfError(f"{name} has {t.numel()} elements, the call writes {n}")


def _need_rows(t, dtype, name, ref, N, P, ld=None):
    """A caller [N, P] int32 buffer written with row stride ld (the ancestors' stride)."""
    _need_cuda(t, dtype, name)
    _same_device(t, ref, name)
    if t.dim() != 2 or t.shape[0] < N or t.shape[1] < P or t.stride(1) != 1:
        raise PfError(f"{name} must be a row-contiguous [>= {N}, >= {P}] tensor, got {tuple(t.shape)}")
    if ld is not None and t.stride(0) != ld:
        raise PfError(f"{name} must have the ancestors' row stride {ld}, got {t.stride(0)}")


def _need_state(X, ref, N, P, batched):
    _same_device(X, ref, "state")
    if batched:
        if X.dim() < 2 or X.shape[0] < N or X.shape[1] < P:
            raise PfError(f"state must be [>= {N}, >= {P}, ...], got {tuple(X.shape)}")
    elif X.dim() < 1 or X.shape[0] < P:
        raise PfError(f"state must have >= {P} rows, got {tuple(X.shape)}")


def _rows(t, name):
    """(ptr, ld) of a 1-D contiguous or 2-D row-strided tensor."""
    if t.dim() == 1:
        if t.stride(0) != 1:
            raise PfError(f"{name} must be contiguous")
        return t.data_ptr(), t.shape[0]
    if t.dim() == 2:
        if t.stride(1) != 1:
            raise PfError(f"{name} rows must be contiguous")
        return t.data_ptr(), t.stride(0)
    raise PfError(f"{name} must be 1-D or 2-D")


def _scheme(s):
    return SCHEMES[s] if isinstance(s, str) else int(s)


def _state_layout(X, batched: bool):
    """(row_bytes, ld_bytes, filter_ld_bytes) of a state tensor [P, ...] or [N, P, ...] whose
    rows (the trailing dims) are contiguous."""
    if not X.is_cuda:
        raise PfError("X must be a CUDA tensor")
    lead = 2 if batched else 1
    if X.dim() < lead:
        raise PfError("state tensor has too few dimensions")
    es = X.element_size()
    inner = X.shape[lead:]
    expect = 1
    for d in range(X.dim() - 1, lead - 1, -1):
        if X.shape[d] != 1 and X.stride(d) != expect:
            raise PfError("state rows (trailing dimensions) must be contiguous")
        expect *= X.shape[d]
    row = es
    for d in inner:
        row *= d
    ld = X.stride(lead - 1) * es
    ldf = X.stride(0) * es if batched else 0
    return row, ld, ldf


def _set_state(opts, state, batched: bool):
    if state is None:
        return
    row, ld, ldf = _state_layout(state, batched)
    opts.state = state.data_ptr()
    opts.state_row_bytes = row
    opts.state_ld_bytes = ld
    opts.state_filter_ld_bytes = ldf


# ----------------------------------------------------------------------------- resamplers
def pf_resample_ex(scheme, logw, seed: int, B: int = 0, ancestors=None, filter_index: int = 0,
                   lse_out=None, normw_out=None, ess_out=None, status_out=None, offspring_out=None,
                   permuted_out=None, flags: int = 0, state=None, workspace=None, stream=None):
    """One filter.  logw: float32 [P] CUDA, or float64 (pf_resample_ex_f64, NS-3d).
    Returns the int32 ancestors tensor.
    workspace: optional device tensor (256-byte aligned, >= pf_workspace_bytes) instead of the pool.
    state: optional [P, ...] tensor gathered in place with the canonical permutation (NS-15/16)."""
    torch = _torch()
    f64 = isinstance(logw, torch.Tensor) and logw.dtype == torch.float64
    _need_cuda(logw, torch.float64 if f64 else torch.float32, "logw")
    if logw.dim() != 1 or logw.stride(0) != 1:
        raise PfError("logw must be a contiguous 1-D tensor")
    P = logw.shape[0]
    if ancestors is None:
        ancestors = torch.empty(P, dtype=torch.int32, device=logw.device)
    _need_vec(ancestors, torch.int32, "ancestors", logw, P)
    opts = _Opts(filter_index=filter_index, flags=flags)
    for name, t, dt, n in (("lse_out", lse_out, torch.float64, 1), ("ess_out", ess_out, torch.float64, 1),
                           ("normw_out", normw_out, torch.float32, P), ("status_out", status_out, torch.int32, 1),
                           ("offspring_out", offspring_out, torch.int32, P),
                           ("permuted_out", permuted_out, torch.int32, P)):
        if t is not None:
            _need_vec(t, dt, name, logw, n)
            setattr(opts, name, t.data_ptr())
    if state is not None:
        _need_state(state, logw, 1, P, False)
    _set_state(opts, state, False)
    _set_workspace(opts, workspace)
    fn = "pf_resample_ex_f64" if f64 else "pf_resample_ex"
    with torch.cuda.device(logw.device):
        rc = getattr(lib(), fn)(_scheme(scheme), logw.data_ptr(), P, seed & (2 ** 64 - 1), B,
                                ancestors.data_ptr(), ctypes.byref(opts), _stream(logw, stream))
    _check(rc, fn)
    return ancestors


def _single(name, scheme):
    def f(logw, seed: int, B: int = 0, ancestors=None, stream=None):
        torch = _torch()
        _need_cuda(logw, torch.float32, "logw")
        if logw.dim() != 1 or logw.stride(0) != 1:
            raise PfError("logw must be a contiguous 1-D tensor")
        P = logw.shape[0]
        if ancestors is None:
            ancestors = torch.empty(P, dtype=torch.int32, device=logw.device)
        _need_vec(ancestors, torch.int32, "ancestors", logw, P)
        with torch.cuda.device(logw.device):
            rc = getattr(lib(), name)(logw.data_ptr(), P, seed & (2 ** 64 - 1), B, ancestors.data_ptr(),
                                      _stream(logw, stream))
        _check(rc, name)
        return ancestors

    f.__name__ = name
    f.__doc__ = f"{name}(logw[P] f32, seed, B, ancestors=None) -> int32 ancestors (scheme {scheme})."
    return f


pf_resample_multinomial = _single("pf_resample_multinomial", "multinomial, Fig. 1(a)")
pf_resample_stratified = _single("pf_resample_stratified", "stratified, Fig. 1(b)")
pf_resample_systematic = _single("pf_resample_systematic", "systematic, Fig. 1(c)")
pf_resample_metropolis = _single("pf_resample_metropolis", "Metropolis, Fig. 1(d), P:128-140")


def pf_resample_batched(scheme, logw, seed: int, B: int = 0, first_filter: int = 0, ancestors=None,
                        lse_out=None, normw_out=None, ess_out=None, status_out=None, offspring_out=None,
                        permuted_out=None, flags: int = 0, state=None, workspace=None, stream=None):
    """N independent filters: logw float32 [N, P] (row-strided) -> int32 ancestors [N, P];
    float64 logw goes through pf_resample_batched_f64 (NS-3d).
    workspace: optional device tensor (256-byte aligned, >= pf_workspace_bytes) instead of the pool.
    state: optional [N, P, ...] tensor gathered in place with the canonical permutation."""
    torch = _torch()
    f64 = isinstance(logw, torch.Tensor) and logw.dtype == torch.float64
    _need_cuda(logw, torch.float64 if f64 else torch.float32, "logw")
    if logw.dim() != 2:
        raise PfError("logw must be [N, P]")
    N, P = logw.shape
    ptr, ld = _rows(logw, "logw")
    if ancestors is None:
        ancestors = torch.empty((N, P), dtype=torch.int32, device=logw.device)
    _need_rows(ancestors, torch.int32, "ancestors", logw, N, P)
    aptr, ald = _rows(ancestors, "ancestors")
    opts = _Opts(flags=flags)
    for name, t, dt, n in (("lse_out", lse_out, torch.float64, N), ("ess_out", ess_out, torch.float64, N),
                           ("normw_out", normw_out, torch.float32, N * P), ("status_out", status_out, torch.int32, N)):
        if t is not None:
            _need_vec(t, dt, name, logw, n)  # dense: [N] / [N, P]
            setattr(opts, name, t.data_ptr())
    for name, t in (("offspring_out", offspring_out), ("permuted_out", permuted_out)):
        if t is not None:
            _need_rows(t, torch.int32, name, logw, N, P, ld=ald)  # written with the ancestors' row stride
            setattr(opts, name, t.data_ptr())
    if state is not None:
        _need_state(state, logw, N, P, True)
    _set_state(opts, state, True)
    _set_workspace(opts, workspace)
    fn = "pf_resample_batched_f64" if f64 else "pf_resample_batched"
    with torch.cuda.device(logw.device):
        rc = getattr(lib(), fn)(_scheme(scheme), ptr, ld, N, P, seed & (2 ** 64 - 1), first_filter, B,
                                aptr, ald, ctypes.byref(opts), _stream(logw, stream))
    _check(rc, fn)
    return ancestors


def pf_workspace_bytes(scheme, N: int, P: int, flags: int = 0, ld_anc: int | None = None) -> int:
    if flags == 0 and ld_anc is None:
        return int(lib().pf_workspace_bytes(_scheme(scheme), N, P))
    return int(lib().pf_workspace_bytes_ex(_scheme(scheme), N, P, flags, P if ld_anc is None else ld_anc))


def _set_workspace(opts, workspace):
    if workspace is None:
        return
    torch = _torch()
    if not isinstance(workspace, torch.Tensor) or not workspace.is_cuda:
        raise PfError("workspace must be a CUDA tensor")
    opts.workspace = workspace.data_ptr()
    opts.workspace_bytes = workspace.numel() * workspace.element_size()


# ----------------------------------------------------------------------------- conversions
def _pair_args(src, src_name, dst, dst_name):
    """(N, P) of a [P] / [N, P] int32 source and a destination of the same shape and device."""
    torch = _torch()
    _need_cuda(src, torch.int32, src_name)
    _need_cuda(dst, torch.int32, dst_name)
    _same_device(dst, src, dst_name)
    if src.dim() == 1:
        _need_vec(dst, torch.int32, dst_name, src, src.shape[0])
        return 1, src.shape[0]
    if src.dim() != 2:
        raise PfError(f"{src_name} must be [P] or [N, P]")
    N, P = src.shape
    _need_rows(dst, torch.int32, dst_name, src, N, P)
    return N, P


def pf_ancestors_to_offspring(anc, offspring=None, stream=None):
    """int32 [P] or [N, P] ancestors -> int32 offspring (NS-14)."""
    torch = _torch()
    _need_cuda(anc, torch.int32, "anc")
    if offspring is None:
        offspring = torch.empty_like(anc)
    N, P = _pair_args(anc, "anc", offspring, "offspring")
    with torch.cuda.device(anc.device):
        if anc.dim() == 1:
            rc = lib().pf_ancestors_to_offspring(anc.data_ptr(), P, offspring.data_ptr(), _stream(anc, stream))
        else:
            ap, ald = _rows(anc, "anc")
            op, old = _rows(offspring, "offspring")
            rc = lib().pf_ancestors_to_offspring_batched(ap, ald, N, P, op, old, _stream(anc, stream))
    _check(rc, "pf_ancestors_to_offspring")
    return offspring


def pf_permute(anc, permuted=None, stream=None):
    """Canonical in-place permutation (NS-15) of int32 [P] or [N, P] ancestors."""
    torch = _torch()
    _need_cuda(anc, torch.int32, "anc")
    if permuted is None:
        permuted = torch.empty_like(anc)
    N, P = _pair_args(anc, "anc", permuted, "permuted")
    with torch.cuda.device(anc.device):
        if anc.dim() == 1:
            rc = lib().pf_permute(anc.data_ptr(), P, permuted.data_ptr(), _stream(anc, stream))
        else:
            ap, ald = _rows(anc, "anc")
            pp, pld = _rows(permuted, "permuted")
            rc = lib().pf_permute_batched(ap, ald, N, P, pp, pld, _stream(anc, stream))
    _check(rc, "pf_permute")
    return permuted


def pf_permute_offspring(offspring, permuted=None, stream=None):
    """Canonical permutation (NS-15) from int32 offspring counts [P] or [N, P] (sum P per row)."""
    torch = _torch()
    _need_cuda(offspring, torch.int32, "offspring")
    if permuted is None:
        permuted = torch.empty_like(offspring)
    N, P = _pair_args(offspring, "offspring", permuted, "permuted")
    with torch.cuda.device(offspring.device):
        if offspring.dim() == 1:
            rc = lib().pf_permute_offspring(offspring.data_ptr(), P, permuted.data_ptr(), _stream(offspring, stream))
        else:
            op, old = _rows(offspring, "offspring")
            pp, pld = _rows(permuted, "permuted")
            rc = lib().pf_permute_offspring_batched(op, old, N, P, pp, pld, _stream(offspring, stream))
    _check(rc, "pf_permute_offspring")
    return permuted


def pf_gather_state(X, permuted, stream=None):
    """In place X[i] <- X[permuted[i]] (NS-16).  X: [P, ...] or [N, P, ...] CUDA tensor with
    contiguous rows; permuted from pf_permute."""
    torch = _torch()
    _need_cuda(permuted, torch.int32, "permuted")
    if permuted.dim() == 1:
        P = permuted.shape[0]
        _need_state(X, permuted, 1, P, False)
        row, ld, _ = _state_layout(X, False)
        with torch.cuda.device(X.device):
            rc = lib().pf_gather_state(X.data_ptr(), row, ld, P, permuted.data_ptr(), _stream(X, stream))
    else:
        N, P = permuted.shape
        _need_state(X, permuted, N, P, True)
        row, ld, ldf = _state_layout(X, True)
        pp, pld = _rows(permuted, "permuted")
        with torch.cuda.device(X.device):
            rc = lib().pf_gather_state_batched(X.data_ptr(), row, ld, ldf, N, P, pp, pld, _stream(X, stream))
    _check(rc, "pf_gather_state")
    return X


def pf_gather_state_out(X, anc, Y=None, stream=None):
    """Out of place Y[i] <- X[anc[i]] for arbitrary ancestors."""
    torch = _torch()
    _need_cuda(anc, torch.int32, "anc")
    if anc.dim() != 1 or not anc.is_contiguous():
        raise PfError("anc must be a contiguous 1-D tensor")
    if Y is None:
        Y = torch.empty_like(X)
    P = anc.shape[0]
    _need_state(X, anc, 1, P, False)
    _need_state(Y, anc, 1, P, False)
    row, ldx, _ = _state_layout(X, False)
    rowy, ldy, _ = _state_layout(Y, False)
    if rowy != row:
        raise PfError("X and Y rows differ in size")
    with torch.cuda.device(X.device):
        rc = lib().pf_gather_state_out(X.data_ptr(), Y.data_ptr(), row, ldx, ldy, P, anc.data_ptr(),
                                       _stream(X, stream))
    _check(rc, "pf_gather_state_out")
    return Y


# ----------------------------------------------------------------------------- giant-filter shards
def _ptr(t):
    return None if t is None else t.data_ptr()


def pf_shard_max(logw_local, stream=None):
    """Stage 1 of a sharded filter: (lmax[1] f32, bad[1] i32) of this shard (device tensors)."""
    torch = _torch()
    _need_cuda(logw_local, torch.float32, "logw")
    lmax = torch.empty(1, dtype=torch.float32, device=logw_local.device)
    bad = torch.empty(1, dtype=torch.int32, device=logw_local.device)
    _check(lib().pf_shard_max(logw_local.data_ptr(), logw_local.shape[0], lmax.data_ptr(), bad.data_ptr(),
                              _stream(logw_local, stream)), "pf_shard_max")
    return lmax, bad


def pf_shard_scan(logw_local, P_global: int, gmax, stream=None):
    """Stage 2: (Q[Pl] u64 as int64 tensor, total[1], wsum[1] f64) with the global max and k_fx(P_global)."""
    torch = _torch()
    _need_cuda(logw_local, torch.float32, "logw")
    Pl = logw_local.shape[0]
    Q = torch.empty(Pl, dtype=torch.int64, device=logw_local.device)
    total = torch.empty(1, dtype=torch.int64, device=logw_local.device)
    wsum = torch.empty(1, dtype=torch.float64, device=logw_local.device)
    _check(lib().pf_shard_scan(logw_local.data_ptr(), Pl, P_global, gmax.data_ptr(), Q.data_ptr(),
                               total.data_ptr(), wsum.data_ptr(), _stream(logw_local, stream)), "pf_shard_scan")
    return Q, total, wsum


def pf_shard_search(scheme, Q, p0: int, P_global: int, totals, shard: int, gmax, gbad, seed: int,
                    filter_index: int, anc_out, stream=None):
    """Stage 3: writes anc_out[k] (int32 [P_global]) for this shard's slots; returns slot_range[2] (int64)."""
    torch = _torch()
    rng = torch.empty(2, dtype=torch.int64, device=Q.device)
    _check(lib().pf_shard_search(_scheme(scheme), Q.data_ptr(), Q.shape[0], p0, P_global, totals.data_ptr(),
                                 totals.shape[0], shard, gmax.data_ptr(), gbad.data_ptr(), seed & (2 ** 64 - 1),
                                 filter_index, anc_out.data_ptr(), rng.data_ptr(), _stream(Q, stream)),
           "pf_shard_search")
    return rng


def pf_shard_route_count(totals, shard: int, P_global: int, gmax, gbad, seed: int, filter_index: int,
                         stream=None):
    """Routed multinomial, stage 3a (include/pf.h): int64 [nshards] positions of this rank's slot
    shard per owner shard."""
    torch = _torch()
    cnt = torch.empty(totals.shape[0], dtype=torch.int64, device=totals.device)
    _check(lib().pf_shard_route_count(totals.data_ptr(), totals.shape[0], shard, P_global, gmax.data_ptr(),
                                      gbad.data_ptr(), seed & (2 ** 64 - 1), filter_index, cnt.data_ptr(),
                                      _stream(totals, stream)), "pf_shard_route_count")
    return cnt


def pf_shard_route_pack(totals, shard: int, P_global: int, gmax, gbad, seed: int, filter_index: int, counts,
                        n_send: int, stream=None):
    """Stage 3b: (x u64 as int64 [n_send], k int32 [n_send]) grouped by owner shard."""
    torch = _torch()
    sx = torch.empty(max(n_send, 1), dtype=torch.int64, device=totals.device)
    sk = torch.empty(max(n_send, 1), dtype=torch.int32, device=totals.device)
    _check(lib().pf_shard_route_pack(totals.data_ptr(), totals.shape[0], shard, P_global, gmax.data_ptr(),
                                     gbad.data_ptr(), seed & (2 ** 64 - 1), filter_index, counts.data_ptr(),
                                     sx.data_ptr(), sk.data_ptr(), _stream(totals, stream)), "pf_shard_route_pack")
    return sx[:n_send], sk[:n_send]


def pf_shard_route_search(Q, p0: int, P_global: int, totals, shard: int, gmax, gbad, recv_x, recv_k, anc_out,
                          stream=None):
    """Stage 3c: anc_out[k] for the received pairs (identity over the shard if the filter is invalid)."""
    n = recv_x.shape[0]
    _check(lib().pf_shard_route_search(Q.data_ptr(), Q.shape[0], p0, P_global, totals.data_ptr(), totals.shape[0],
                                       shard, gmax.data_ptr(), gbad.data_ptr(), recv_x.data_ptr() if n else None,
                                       recv_k.data_ptr() if n else None, n, anc_out.data_ptr(), _stream(Q, stream)),
           "pf_shard_route_search")
    return anc_out


def pf_shard_spacings_total(P_global: int, nshards: int, shard: int, seed: int, filter_index: int, device,
                            stream=None):
    """Stage 2b (sorted multinomial, NS-12): etotal[1] (u64 as int64) = sum of the spacings
    e_k over spacing shard ``shard`` of ``nshards`` (include/pf.h)."""
    torch = _torch()
    et = torch.empty(1, dtype=torch.int64, device=device)
    _check(lib().pf_shard_spacings_total(P_global, nshards, shard, seed & (2 ** 64 - 1), filter_index,
                                         et.data_ptr(), _stream(et, stream)), "pf_shard_spacings_total")
    return et


def pf_shard_search_sorted_workspace_bytes(P_global: int) -> int:
    return int(lib().pf_shard_search_sorted_workspace_bytes(P_global))


def pf_shard_search_sorted(Q, p0: int, P_global: int, totals, etotals, shard: int, gmax, gbad, seed: int,
                           filter_index: int, anc_out, workspace=None, stream=None):
    """Stage 3 of the sharded sorted multinomial: writes anc_out[k] (int32 [P_global]) for this
    shard's slots; returns slot_range[2] (int64).  workspace: optional uint8 device tensor."""
    torch = _torch()
    rng = torch.zeros(2, dtype=torch.int64, device=Q.device)
    wp, wb = (workspace.data_ptr(), workspace.numel() * workspace.element_size()) if workspace is not None else (None, 0)
    _check(lib().pf_shard_search_sorted(Q.data_ptr(), Q.shape[0], p0, P_global, totals.data_ptr(),
                                        etotals.data_ptr(), totals.shape[0], shard, gmax.data_ptr(), gbad.data_ptr(),
                                        seed & (2 ** 64 - 1), filter_index, anc_out.data_ptr(), rng.data_ptr(), wp,
                                        wb, _stream(Q, stream)), "pf_shard_search_sorted")
    return rng


def pf_shard_weights(logw_local, gmax, w_out=None, stream=None):
    torch = _torch()
    _need_cuda(logw_local, torch.float32, "logw")
    if w_out is None:
        w_out = torch.empty_like(logw_local)
    _check(lib().pf_shard_weights(logw_local.data_ptr(), logw_local.shape[0], gmax.data_ptr(), w_out.data_ptr(),
                                  _stream(logw_local, stream)), "pf_shard_weights")
    return w_out


def pf_metropolis_from_weights(w_full, slot0: int, nslots: int, seed: int, B: int, filter_index: int = 0,
                               gmax=None, gbad=None, anc=None, stream=None):
    torch = _torch()
    _need_cuda(w_full, torch.float32, "w_full")
    if anc is None:
        anc = torch.empty(nslots, dtype=torch.int32, device=w_full.device)
    _check(lib().pf_metropolis_from_weights(w_full.data_ptr(), w_full.shape[0], slot0, nslots,
                                            seed & (2 ** 64 - 1), B, filter_index, _ptr(gmax), _ptr(gbad),
                                            anc.data_ptr(), _stream(w_full, stream)), "pf_metropolis_from_weights")
    return anc


# ----------------------------------------------------------------------------- particle migration
def pf_shard_offspring(anc, win0: int, Pw: int, slot_range=None, gmax=None, gbad=None, out=None, stream=None):
    """Stage 4a: offspring[Pw] (int32) of particles [win0, win0 + Pw) from the global ancestors in
    ``anc`` (entries slot_range[0]..slot_range[1], or all of them when slot_range is None)."""
    torch = _torch()
    _need_cuda(anc, torch.int32, "anc")
    if out is None:
        out = torch.empty(Pw, dtype=torch.int32, device=anc.device)
    _check(lib().pf_shard_offspring(anc.data_ptr(), anc.shape[0], _ptr(slot_range), win0, Pw, _ptr(gmax),
                                    _ptr(gbad), out.data_ptr(), _stream(anc, stream)), "pf_shard_offspring")
    return out


def pf_shard_migration_counts(offspring, stream=None):
    """Stage 4b: (counts int64[2] device {E extras, F free slots}, plan) of the shard; the plan
    (device bytes) feeds pf_shard_migrate_pack / _unpack of the same offspring."""
    torch = _torch()
    _need_cuda(offspring, torch.int32, "offspring")
    Pl = offspring.shape[0]
    c = torch.empty(2, dtype=torch.int64, device=offspring.device)
    plan = torch.empty(max(1, lib().pf_shard_migration_plan_bytes(Pl) // 8), dtype=torch.int64,
                       device=offspring.device)
    _check(lib().pf_shard_migration_counts(offspring.data_ptr(), Pl, plan.data_ptr(), c.data_ptr(),
                                           _stream(offspring, stream)), "pf_shard_migration_counts")
    return c, plan


def _rows_view(X):
    if X is None:
        return 0, 0
    row, ld, _ = _state_layout(X, False)
    return row, ld


def pf_shard_migrate_pack(X, offspring, plan, p0: int, E: int, stream=None):
    """Stage 4c: (send_rows uint8 [E, row_bytes] or None, send_src int32 [E]) — the shard's
    extras in NS-15 order.  E = this shard's extras count (pf_shard_migration_counts)."""
    torch = _torch()
    _need_cuda(offspring, torch.int32, "offspring")
    dev = offspring.device
    row, ld = _rows_view(X)
    src = torch.empty(max(E, 1), dtype=torch.int32, device=dev)
    rows = torch.empty((max(E, 1), row), dtype=torch.uint8, device=dev) if row else None
    _check(lib().pf_shard_migrate_pack(_ptr(X), row, ld, offspring.shape[0], p0, offspring.data_ptr(),
                                       plan.data_ptr(), _ptr(rows), src.data_ptr(), _stream(offspring, stream)),
           "pf_shard_migrate_pack")
    return (rows[:E] if rows is not None else None), src[:E]


def pf_shard_migrate_unpack(X, offspring, plan, p0: int, recv_rows, recv_src, perm_out=None, stream=None):
    """Stage 4d: free slots of X (in place) <- recv_rows; returns perm_out (int32 [Pl]) when
    recv_src is given: the global index of the particle each slot now holds."""
    torch = _torch()
    _need_cuda(offspring, torch.int32, "offspring")
    row, ld = _rows_view(X)
    if perm_out is None and recv_src is not None:
        perm_out = torch.empty(offspring.shape[0], dtype=torch.int32, device=offspring.device)
    if recv_rows is not None and recv_rows.numel() == 0:
        recv_rows = None
    if row and recv_rows is not None and (recv_rows.dim() != 2 or recv_rows.shape[1] != row):
        raise PfError("recv_rows must be [F, row_bytes] uint8")
    _check(lib().pf_shard_migrate_unpack(_ptr(X), row, ld, offspring.shape[0], p0, offspring.data_ptr(),
                                         plan.data_ptr(), _ptr(recv_rows), _ptr(recv_src), _ptr(perm_out),
                                         _stream(offspring, stream)), "pf_shard_migrate_unpack")
    return perm_out


# ----------------------------------------------------------------------------- C4 demo model
def pf_lg_init(X, phi: float, sigma_x: float, seed: int, stream=None):
    torch = _torch()
    _need_cuda(X, torch.float32, "X")
    _check(lib().pf_lg_init(X.data_ptr(), X.stride(0), X.shape[0], X.shape[1], phi, sigma_x, seed & (2 ** 64 - 1),
                            _stream(X, stream)), "pf_lg_init")
    return X


def pf_lg_propagate_weight(X, phi: float, sigma_x: float, sigma_y: float, y: float, seed: int, t: int, logw=None,
                           stream=None):
    torch = _torch()
    _need_cuda(X, torch.float32, "X")
    if logw is None:
        logw = torch.empty(X.shape[0], dtype=torch.float32, device=X.device)
    _check(lib().pf_lg_propagate_weight(X.data_ptr(), X.stride(0), X.shape[0], X.shape[1], phi, sigma_x, sigma_y,
                                        float(y), seed & (2 ** 64 - 1), t, logw.data_ptr(), _stream(X, stream)),
           "pf_lg_propagate_weight")
    return logw


def pf_lg_accumulate(lse, P: int, sigma_y: float, loglik, stream=None):
    _check(lib().pf_lg_accumulate(lse.data_ptr(), P, sigma_y, loglik.data_ptr(), _stream(lse, stream)),
           "pf_lg_accumulate")
    return loglik


# ----------------------------------------------------------------------------- host helpers
def pf_metropolis_required_B(P: int, w_max: float, eps: float) -> int:
    """Eq. (5), alpha Eq. (2), beta = 1/P."""
    return int(lib().pf_metropolis_required_B(P, w_max, eps))


def pf_launch_count() -> int:
    return int(lib().pf_launch_count())


def pf_status_string(status: int) -> str:
    return lib().pf_status_string(int(status)).decode()


class _KernelTime(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_uint64), ("total_ms", ctypes.c_double),
                ("alg_bytes", ctypes.c_uint64), ("row_bytes", ctypes.c_uint64)]


def pf_profile_enable(on: bool = True) -> None:
    """Bracket every kernel launch with CUDA events on its own stream (tracing)."""
    lib().pf_profile_enable(1 if on else 0)


def pf_profile_collect() -> dict:
    """{kernel name: (launches, total_ms, alg_bytes, row_bytes)} since the last collect (waits for
    the events).  alg_bytes: summed algorithmic HBM bytes of those launches as stated by the
    library (0 = not stated); row_bytes: summed bytes per moved state row (multiply by the rows
    the gather moved)."""
    buf = (_KernelTime * 64)()
    n = lib().pf_profile_collect(buf, 64)
    if n < 0:
        raise PfError("pf_profile_collect: CUDA error")
    return {buf[i].name.decode(): (int(buf[i].launches), float(buf[i].total_ms), int(buf[i].alg_bytes),
                                   int(buf[i].row_bytes)) for i in range(min(n, 64))}


def pf_set_fusion(on: bool = True) -> None:
    """Diagnostics: False forces the multi-launch paths everywhere (identical results)."""
    lib().pf_set_fusion(1 if on else 0)


def pf_version() -> str:
    return lib().pf_version().decode()


def pf_release() -> None:
    lib().pf_release()
