"""CPU oracle for the resampling hot path of arXiv 1202.6163 — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_1202_6163_b200``) never imports it and shares no code with it.

This module is argument marshalling (numpy <-> ctypes) around ``liboracle.so``,
which is plain single-threaded C (``pfo.c``) written step by step from
PAPER.md and the numeric spec in DESIGN.md §3.  Every function cites the
passage it follows in ``pfo.c``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

MULTINOMIAL, STRATIFIED, SYSTEMATIC, METROPOLIS = 1, 2, 3, 4
SCHEMES = {"multinomial": 1, "stratified": 2, "systematic": 3, "metropolis": 4}
FILTER_OK, FILTER_INVALID = 0, 1

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, IEEE-exact flags)."""
    src = os.path.join(_HERE, "pfo.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "pfo.h"))
    ):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, src, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i32, u32, i64, u64, f32, f64 = (ctypes.c_int32, ctypes.c_uint32, ctypes.c_int64,
                                        ctypes.c_uint64, ctypes.c_float, ctypes.c_double)
        L.pfo_philox4x32_10.argtypes = [P, P, P]
        L.pfo_dexp.argtypes = [f32]
        L.pfo_dexp.restype = f32
        L.pfo_lmax.argtypes = [P, i32, P]
        L.pfo_weights.argtypes = [P, i32, P]
        L.pfo_kfx.argtypes = [i32]
        L.pfo_weights_with.argtypes = [P, i32, f32, P]
        L.pfo_cumulative_with.argtypes = [P, i32, f32, ctypes.c_int, P]
        L.pfo_cumulative.argtypes = [P, i32, P]
        L.pfo_position.argtypes = [ctypes.c_int, i32, u64, u64, u32, i64]
        L.pfo_position.restype = u64
        L.pfo_upper_bound.argtypes = [P, i32, u64]
        L.pfo_upper_bound.restype = i32
        L.pfo_systematic_from_R.argtypes = [P, i32, u64, P]
        L.pfo_metropolis_chains.argtypes = [P, i32, i64, i32, u64, i32, u32, P]
        L.pfo_resample.argtypes = [ctypes.c_int, P, i32, u64, i32, u32, P, P, P, P]
        L.pfo_resample_batched.argtypes = [ctypes.c_int, P, i64, i32, i32, u64, u32, i32, P, i64, P]
        L.pfo_ancestors_to_offspring.argtypes = [P, i32, P]
        L.pfo_offspring_to_ancestors.argtypes = [P, i32, P]
        L.pfo_permute.argtypes = [P, i32, P]
        L.pfo_gather_inplace.argtypes = [P, i64, i64, i32, P]
        L.pfo_gather_out.argtypes = [P, P, i64, i64, i64, i32, P]
        L.pfo_dlog.argtypes = [f64]
        L.pfo_dlog.restype = f64
        L.pfo_spacing.argtypes = [u64, u32, i64]
        L.pfo_spacing.restype = u64
        L.pfo_spacings.argtypes = [i32, u64, u32, P]
        L.pfo_resample_sorted_multinomial.argtypes = [P, i32, u64, u32, P]
        L.pfo_shift_f64.argtypes = [P, i32, P, P]
        L.pfo_resample_f64.argtypes = [ctypes.c_int, ctypes.c_int, P, i32, u64, i32, u32, P, P, P, P]
        L.pfo_resample_sorted_weights.argtypes = [ctypes.c_int, P, i32, u64, u32, P, P, P, P]
        L.pfo_metropolis_required_B.argtypes = [i64, f64, f64]
        L.pfo_metropolis_required_B.restype = i32
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _scheme(s):
    return SCHEMES[s] if isinstance(s, str) else int(s)


def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().pfo_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def dexp(t: float) -> float:
    return float(lib().pfo_dexp(float(t)))


def dexp_array(t: np.ndarray) -> np.ndarray:
    f = lib().pfo_dexp
    return np.array([f(float(v)) for v in np.asarray(t, dtype=np.float32)], dtype=np.float32)


def lmax(logw: np.ndarray):
    logw = np.ascontiguousarray(logw, dtype=np.float32)
    out = ctypes.c_float()
    st = lib().pfo_lmax(_p(logw), len(logw), ctypes.byref(out))
    return st, out.value


def weights(logw: np.ndarray):
    logw = np.ascontiguousarray(logw, dtype=np.float32)
    w = np.zeros(len(logw), dtype=np.float32)
    st = lib().pfo_weights(_p(logw), len(logw), _p(w))
    return st, w


def weights_with(logw: np.ndarray, lmax: float) -> np.ndarray:
    logw = np.ascontiguousarray(logw, dtype=np.float32)
    w = np.zeros(len(logw), dtype=np.float32)
    lib().pfo_weights_with(_p(logw), len(logw), float(lmax), _p(w))
    return w


def cumulative_with(logw: np.ndarray, lmax: float, kfx_bits: int) -> np.ndarray:
    logw = np.ascontiguousarray(logw, dtype=np.float32)
    Q = np.zeros(len(logw), dtype=np.uint64)
    lib().pfo_cumulative_with(_p(logw), len(logw), float(lmax), int(kfx_bits), _p(Q))
    return Q


def kfx(P: int) -> int:
    return int(lib().pfo_kfx(P))


def cumulative(logw: np.ndarray):
    logw = np.ascontiguousarray(logw, dtype=np.float32)
    Q = np.zeros(len(logw), dtype=np.uint64)
    st = lib().pfo_cumulative(_p(logw), len(logw), _p(Q))
    return st, Q


def position(scheme, P, Qtot, seed, filter_index, k) -> int:
    return int(lib().pfo_position(_scheme(scheme), P, Qtot, seed, filter_index, k))


def upper_bound(Q: np.ndarray, x: int) -> int:
    Q = np.ascontiguousarray(Q, dtype=np.uint64)
    return int(lib().pfo_upper_bound(_p(Q), len(Q), x))


def systematic_from_R(Q: np.ndarray, R: int) -> np.ndarray:
    Q = np.ascontiguousarray(Q, dtype=np.uint64)
    a = np.zeros(len(Q), dtype=np.int32)
    lib().pfo_systematic_from_R(_p(Q), len(Q), R, _p(a))
    return a


def metropolis_chains(w: np.ndarray, slot0: int, nslots: int, seed: int, B: int, filter_index: int = 0,
                      P: int | None = None):
    w = np.ascontiguousarray(w, dtype=np.float32)
    a = np.zeros(nslots, dtype=np.int32)
    lib().pfo_metropolis_chains(_p(w), len(w) if P is None else P, slot0, nslots, seed, B, filter_index, _p(a))
    return a


def resample(scheme, logw: np.ndarray, seed: int, B: int = 0, filter_index: int = 0, side: bool = False):
    """Returns (status, ancestors[, lse, normw, ess])."""
    logw = np.ascontiguousarray(logw, dtype=np.float32)
    P = len(logw)
    a = np.zeros(P, dtype=np.int32)
    if side:
        lse = ctypes.c_double()
        ess = ctypes.c_double()
        v = np.zeros(P, dtype=np.float32)
        st = lib().pfo_resample(_scheme(scheme), _p(logw), P, seed, B, filter_index, _p(a),
                                ctypes.byref(lse), _p(v), ctypes.byref(ess))
        return st, a, lse.value, v, ess.value
    st = lib().pfo_resample(_scheme(scheme), _p(logw), P, seed, B, filter_index, _p(a), None, None, None)
    return st, a


def resample_batched(scheme, logw: np.ndarray, seed: int, B: int = 0, first_filter: int = 0):
    logw = np.ascontiguousarray(logw, dtype=np.float32)
    N, P = logw.shape
    a = np.zeros((N, P), dtype=np.int32)
    st = np.zeros(N, dtype=np.int32)
    lib().pfo_resample_batched(_scheme(scheme), _p(logw), P, N, P, seed, first_filter, B, _p(a), P, _p(st))
    return st, a


def shift_f64(logw: np.ndarray):
    """NS-3d (R-21): (status, t float32[P], lmax float64) of binary64 log-weights."""
    logw = np.ascontiguousarray(logw, dtype=np.float64)
    t = np.zeros(len(logw), dtype=np.float32)
    lm = ctypes.c_double()
    st = lib().pfo_shift_f64(_p(logw), len(logw), _p(t), ctypes.byref(lm))
    return st, t, lm.value


def resample_f64(scheme, logw: np.ndarray, seed: int, B: int = 0, filter_index: int = 0, side: bool = False,
                 sorted: bool = False):
    """binary64 log-weights (NS-3d): returns (status, ancestors[, lse, normw, ess])."""
    logw = np.ascontiguousarray(logw, dtype=np.float64)
    P = len(logw)
    a = np.zeros(P, dtype=np.int32)
    lse, ess = ctypes.c_double(), ctypes.c_double()
    v = np.zeros(P, dtype=np.float32)
    st = lib().pfo_resample_f64(_scheme(scheme), int(sorted), _p(logw), P, seed, B, filter_index, _p(a),
                                ctypes.byref(lse) if side else None, _p(v) if side else None,
                                ctypes.byref(ess) if side else None)
    if side:
        return st, a, lse.value, v, ess.value
    return st, a


def resample_sorted_weights(scheme, logw: np.ndarray, seed: int, filter_index: int = 0, side: bool = False):
    """NS-17 pre-sorted weights: returns (status, ancestors[, lse, normw, ess])."""
    logw = np.ascontiguousarray(logw, dtype=np.float32)
    P = len(logw)
    a = np.zeros(P, dtype=np.int32)
    lse, ess = ctypes.c_double(), ctypes.c_double()
    v = np.zeros(P, dtype=np.float32)
    st = lib().pfo_resample_sorted_weights(_scheme(scheme), _p(logw), P, seed, filter_index, _p(a),
                                           ctypes.byref(lse) if side else None, _p(v) if side else None,
                                           ctypes.byref(ess) if side else None)
    if side:
        return st, a, lse.value, v, ess.value
    return st, a


def dlog(x: float) -> float:
    return float(lib().pfo_dlog(float(x)))


def spacings(P: int, seed: int, filter_index: int = 0) -> np.ndarray:
    G = np.zeros(P + 1, dtype=np.uint64)
    lib().pfo_spacings(P, seed, filter_index, _p(G))
    return G


def resample_sorted_multinomial(logw: np.ndarray, seed: int, filter_index: int = 0):
    logw = np.ascontiguousarray(logw, dtype=np.float32)
    a = np.zeros(len(logw), dtype=np.int32)
    st = lib().pfo_resample_sorted_multinomial(_p(logw), len(logw), seed, filter_index, _p(a))
    return st, a


def ancestors_to_offspring(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.int32)
    o = np.zeros(len(a), dtype=np.int32)
    lib().pfo_ancestors_to_offspring(_p(a), len(a), _p(o))
    return o


def offspring_to_ancestors(o: np.ndarray) -> np.ndarray:
    o = np.ascontiguousarray(o, dtype=np.int32)
    a = np.zeros(len(o), dtype=np.int32)
    lib().pfo_offspring_to_ancestors(_p(o), len(o), _p(a))
    return a


def permute(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.int32)
    p = np.zeros(len(a), dtype=np.int32)
    lib().pfo_permute(_p(a), len(a), _p(p))
    return p


def gather_inplace(X: np.ndarray, perm: np.ndarray) -> np.ndarray:
    X = np.ascontiguousarray(X).copy()
    perm = np.ascontiguousarray(perm, dtype=np.int32)
    rb = X.strides[0]
    lib().pfo_gather_inplace(_p(X), rb, rb, len(perm), _p(perm))
    return X


def gather_out(X: np.ndarray, anc: np.ndarray) -> np.ndarray:
    X = np.ascontiguousarray(X)
    Y = np.empty_like(X)
    anc = np.ascontiguousarray(anc, dtype=np.int32)
    rb = X.strides[0]
    lib().pfo_gather_out(_p(X), _p(Y), rb, rb, rb, len(anc), _p(anc))
    return Y


def required_B(P: int, w_max: float, eps: float) -> int:
    return int(lib().pfo_metropolis_required_B(P, w_max, eps))
