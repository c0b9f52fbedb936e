"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes/numpy wrapper around ``oracle/liboracle.so`` (compiled from ``sp_oracle.c`` by
``__graft_entry__.build()`` or :func:`build`).  The oracle is a plain, slow CPU reference written
from PAPER.md (arXiv 2605.05219); see ``sp_oracle.c`` for the passage each function follows.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs (``cpu_baseline`` and
``--impl reference``) may import this module.  The CUDA product path
(``paper_2605_05219_b200``) never imports it and shares no code with it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_c_int, _c_i32, _c_i64 = ctypes.c_int, ctypes.c_int32, ctypes.c_int64
_vp = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (-O2, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-pthread",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.or_lcp_hist.argtypes = [_i32p, _i64p, _c_i32, _i32p, _i64p, _i32p, _c_i64, _c_i32,
                                  _i32p, _vp, _c_int]
        L.or_prefix.argtypes = [_i64p, _c_i32, _i64p, _i64p]
        L.or_dp_naive.argtypes = [_i64p, _c_i32, _c_i32, _i64p, _i32p]
        L.or_dp_cht.argtypes = [_i64p, _c_i32, _c_i32, _i64p, _i32p]
        L.or_backtrack.argtypes = [_i32p, _i64p, _c_i32, _c_i32, _i32p]
        L.or_expected_cost.argtypes = [_i64p, _c_i32, _i32p, _c_i32]
        L.or_expected_cost.restype = ctypes.c_int64
        L.or_worst_case.argtypes = [_c_i32, _i32p, _c_i32]
        L.or_worst_case.restype = ctypes.c_int32
        L.or_brute_force.argtypes = [_i64p, _c_i32, _c_i32, _i32p, ctypes.POINTER(_c_i32),
                                     ctypes.POINTER(_c_i64)]
        L.or_balanced.argtypes = [_c_i32, _c_i32, _i32p]
        L.or_block.argtypes = [_c_i32, _c_i32, _i32p]
        L.or_dp_naive_f64.argtypes = [_f64p, _c_i32, _c_i32, _f64p, _i32p]
        L.or_expected_cost_f64.argtypes = [_f64p, _c_i32, _i32p, _c_i32]
        L.or_expected_cost_f64.restype = ctypes.c_double
        L.or_dp_grid_naive.argtypes = [_i64p, _c_i32, _c_i32, _c_i32, _i64p, _i32p]
        L.or_clip_to_blocks.argtypes = [_i32p, _c_i32, _c_i32, _i32p]
        L.or_sqrt_positions.argtypes = [_c_i32, _i32p]
        L.or_log_positions.argtypes = [_c_i32, _c_i32, _i32p]
        L.or_match_longest_prefix.argtypes = [_i32p, _i64p, _c_i32, _vp, _i32p, _i64p, _c_i64,
                                              _i32p, _i32p]
        L.or_gamma_hist.argtypes = [_i32p, _c_i64, _c_i32, ctypes.c_double, _f64p]
        L.or_gamma_variance_term.argtypes = [ctypes.c_double, _c_i64, _c_i32]
        L.or_gamma_variance_term.restype = ctypes.c_double
        L.or_place_batch.argtypes = [_i32p, _c_i32, _c_i32, _c_i32, _c_int, _i32p, _i32p, _i64p,
                                     _vp, _c_int]
        L.or_eval_batch.argtypes = [_i32p, _c_i32, _c_i32, _i32p, _i32p, _c_i32, _c_i32, _c_int,
                                    _i64p, _vp, _c_int]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _counts(c) -> np.ndarray:
    c = np.ascontiguousarray(np.asarray(c, dtype=np.int64))
    assert c.ndim == 1 and c.size >= 2, "counts must be c[0..N] (bin 0 = miss)"
    return c


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"oracle {what} failed with code {rc}")


def lcp_hist(entry_tokens, entry_off, req_tokens, req_off, req_entry, N, n_entries=None,
             hist=None, nthreads=1):
    entry_tokens = np.ascontiguousarray(entry_tokens, dtype=np.int32)
    entry_off = np.ascontiguousarray(entry_off, dtype=np.int64)
    req_tokens = np.ascontiguousarray(req_tokens, dtype=np.int32)
    req_off = np.ascontiguousarray(req_off, dtype=np.int64)
    req_entry = np.ascontiguousarray(req_entry, dtype=np.int32)
    E = len(entry_off) - 1 if n_entries is None else n_entries
    R = len(req_off) - 1
    if hist is None:
        hist = np.zeros((E, N + 1), dtype=np.int32)
    lcp = np.zeros(R, dtype=np.int32)
    _check(lib().or_lcp_hist(entry_tokens, entry_off, E, req_tokens, req_off, req_entry, R, N,
                             hist, _ptr(lcp), nthreads), "lcp_hist")
    return hist, lcp


def prefix(c):
    c = _counts(c)
    N = c.size - 1
    P = np.zeros(N + 1, np.int64)
    T = np.zeros(N + 1, np.int64)
    _check(lib().or_prefix(c, N, P, T), "prefix")
    return P, T


def dp(c, M, algo="naive"):
    """Return (dp[M+1][N+1] int64, opt[M+1][N+1] int32)."""
    c = _counts(c)
    N = c.size - 1
    D = np.zeros((M + 1) * (N + 1), np.int64)
    O = np.zeros((M + 1) * (N + 1), np.int32)
    fn = lib().or_dp_naive if algo == "naive" else lib().or_dp_cht
    _check(fn(c, N, M, D, O), f"dp_{algo}")
    return D.reshape(M + 1, N + 1), O.reshape(M + 1, N + 1)


def backtrack(opt, c, M):
    c = _counts(c)
    N = c.size - 1
    P, _ = prefix(c)
    pos = np.zeros(max(M, 1), np.int32)
    k = lib().or_backtrack(np.ascontiguousarray(opt, dtype=np.int32).ravel(), P, N, M, pos)
    return pos[:k].copy()


def place(c, M, algo="naive"):
    """Rule-B placement: (positions ascending, cost V_M = dp[M][N], V_0..V_M)."""
    D, O = dp(c, M, algo)
    pos = backtrack(O, c, M)
    return pos, int(D[M, -1]), D[:, -1].copy()


def expected_cost(c, pos):
    c = _counts(c)
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    return int(lib().or_expected_cost(c, c.size - 1, pos if pos.size else np.zeros(1, np.int32),
                                      pos.size))


def worst_case(N, pos):
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    return int(lib().or_worst_case(N, pos if pos.size else np.zeros(1, np.int32), pos.size))


def brute_force(c, M):
    c = _counts(c)
    N = c.size - 1
    pos = np.zeros(max(M, 1), np.int32)
    k = _c_i32(0)
    cost = _c_i64(0)
    _check(lib().or_brute_force(c, N, M, pos, ctypes.byref(k), ctypes.byref(cost)), "brute")
    return pos[:k.value].copy(), int(cost.value)


def balanced(N, M):
    pos = np.zeros(max(M, 1), np.int32)
    k = lib().or_balanced(N, M, pos)
    if k < 0:
        raise ValueError("balanced: bad N/M")
    return pos[:k].copy()


def block(N, B):
    pos = np.zeros(max(N // max(B, 1), 1), np.int32)
    k = lib().or_block(N, B, pos)
    if k < 0:
        raise ValueError("block: bad N/B")
    return pos[:k].copy()


def dp_f64(w, M):
    w = np.ascontiguousarray(w, dtype=np.float64)
    N = w.size - 1
    D = np.zeros((M + 1) * (N + 1), np.float64)
    O = np.zeros((M + 1) * (N + 1), np.int32)
    _check(lib().or_dp_naive_f64(w, N, M, D, O), "dp_f64")
    return D.reshape(M + 1, N + 1), O.reshape(M + 1, N + 1)


def expected_cost_f64(w, pos):
    w = np.ascontiguousarray(w, dtype=np.float64)
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    return float(lib().or_expected_cost_f64(w, w.size - 1,
                                            pos if pos.size else np.zeros(1, np.int32), pos.size))


def place_batch(hist, M, algo="cht", nthreads=1, with_budget=False):
    hist = np.ascontiguousarray(hist, dtype=np.int32)
    E, W = hist.shape
    N = W - 1
    pos = np.zeros((E, max(M, 1)), np.int32)
    npos = np.zeros(E, np.int32)
    cost = np.zeros(E, np.int64)
    cbb = np.zeros((E, M + 1), np.int64) if with_budget else None
    _check(lib().or_place_batch(hist, E, N, M, 0 if algo == "naive" else 1, pos, npos, cost,
                                _ptr(cbb), nthreads), "place_batch")
    return pos[:, :M], npos, cost, cbb


def eval_batch(hist, positions, n_positions, broadcast=True, nthreads=1):
    hist = np.ascontiguousarray(hist, dtype=np.int32)
    positions = np.ascontiguousarray(positions, dtype=np.int32)
    n_positions = np.ascontiguousarray(n_positions, dtype=np.int32)
    E, W = hist.shape
    S, max_pos = (positions.shape[0], positions.shape[1]) if broadcast else \
        (positions.shape[1], positions.shape[2])
    cost = np.zeros((E, S), np.int64)
    worst = np.zeros((E, S), np.int32)
    _check(lib().or_eval_batch(hist, E, W - 1, positions, n_positions, S, max_pos,
                               1 if broadcast else 0, cost, _ptr(worst), nthreads), "eval_batch")
    return cost, worst


def place_grid(c, M, B):
    """Block-restricted DP (S:206-214 candidate_grid): positions in multiples of B.  Backtrack:
    leftmost argmin, stopping as soon as no checkpoint improves the remaining prefix
    (dp[m][j] == dp[0][j] = T_j) -- the colex-minimal optimum; for the unrestricted DP this is
    exactly rule B's P_j = 0 stop (reading R13)."""
    c = _counts(c)
    N = c.size - 1
    D = np.zeros((M + 1) * (N + 1), np.int64)
    O = np.zeros((M + 1) * (N + 1), np.int32)
    _check(lib().or_dp_grid_naive(c, N, M, B, D, O), "dp_grid")
    D, O = D.reshape(M + 1, N + 1), O.reshape(M + 1, N + 1)
    P, _ = prefix(c)
    pos, j, m = [], N, M
    while m > 0 and D[m, j] < D[0, j]:
        s = int(O[m, j])
        pos.append(s)
        j, m = s - 1, m - 1
    return np.asarray(pos[::-1], np.int32), int(D[M, N]), D[:, N].copy()


def clip_to_blocks(pos, B):
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    out = np.zeros(max(pos.size, 1), np.int32)
    k = lib().or_clip_to_blocks(pos if pos.size else np.zeros(1, np.int32), pos.size, B, out)
    return out[:k].copy()


def sqrt_positions(N):
    out = np.zeros(N, np.int32)
    return out[:lib().or_sqrt_positions(N, out)].copy()


def log_positions(N, M):
    out = np.zeros(max(M, 1), np.int32)
    k = lib().or_log_positions(N, M, out)
    if k < 0:
        raise ValueError("log_positions: bad N/M")
    return out[:k].copy()


def gamma_hist(depths, N, gamma):
    """f2: Thm 4's exponentially weighted histogram of the depth stream (definition)."""
    d = np.ascontiguousarray(depths, dtype=np.int32)
    p = np.zeros(N + 1, np.float64)
    _check(lib().or_gamma_hist(d if d.size else np.zeros(1, np.int32), d.size, N, gamma, p),
           "or_gamma_hist")
    return p


def gamma_variance_term(gamma, t, N):
    return lib().or_gamma_variance_term(gamma, t, N)


def match_longest_prefix(entry_tokens, entry_off, req_tokens, req_off, insertion=None):
    """f4: (match_entry [R] int32, -1 = none; match_depth [R] int32) by brute force."""
    et = np.ascontiguousarray(entry_tokens, dtype=np.int32)
    eo = np.ascontiguousarray(entry_off, dtype=np.int64)
    rt = np.ascontiguousarray(req_tokens, dtype=np.int32)
    ro = np.ascontiguousarray(req_off, dtype=np.int64)
    E, R = eo.size - 1, ro.size - 1
    me = np.zeros(max(R, 1), np.int32)
    md = np.zeros(max(R, 1), np.int32)
    ins = None if insertion is None else np.ascontiguousarray(insertion, dtype=np.int64)
    _check(lib().or_match_longest_prefix(et if et.size else np.zeros(1, np.int32), eo, E,
                                         _ptr(ins) if ins is not None else None,
                                         rt if rt.size else np.zeros(1, np.int32), ro, R, me, md),
           "or_match_longest_prefix")
    return me[:R].copy(), md[:R].copy()
