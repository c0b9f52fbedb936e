"""Thin ctypes binding of libsparseprefix.so (include/sparse_prefix.h), same names as the C ABI.

Argument marshalling only: every step of the hot path runs in the CUDA kernels of the library.
There is no CPU fallback -- if the library is missing or a tensor is not on a CUDA device, the
call raises.  torch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SP_LIB") or os.path.join(_HERE, "libsparseprefix.so")

SP_OK = 0
SP_ERR_BAD_LENGTH = 1
SP_ERR_BUDGET_TOO_LARGE = 2
SP_ERR_BAD_ARGUMENT = 3
SP_ERR_OVERFLOW = 4
SP_ERR_BAD_POSITIONS = 5
SP_ERR_WORKSPACE = 6
SP_ERR_CUDA = 7
SP_ERR_INTERNAL = 8

# comparison / test hooks (sp_debug_set)
SP_DBG_NO_HULL, SP_DBG_HULL_LEAN, SP_DBG_HULL_SPLIT = 0, 1, 2
SP_DBG_HULL_LOGCAP, SP_DBG_HULL_NO_ORDER, SP_DBG_EVAL_PATH = 3, 4, 5

SP_W_COUNTS_I32 = 0
SP_W_COUNTS_I64 = 1
SP_W_PROB_F64 = 2
SP_MAX_N = 65535

_WTYPE = {torch.int32: SP_W_COUNTS_I32, torch.int64: SP_W_COUNTS_I64,
          torch.float64: SP_W_PROB_F64}

_lib = None
_vp, _i32, _i64, _sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t

SYMBOLS = {
    # name: (restype, argtypes)
    "sp_overlap_hist": (ctypes.c_int, [_vp, _vp, _i32, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp]),
    "sp_accumulate_depths": (ctypes.c_int, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp]),
    "sp_place_checkpoints_workspace_bytes": (_sz, [_i32, _i32, _i32]),
    "sp_place_checkpoints": (ctypes.c_int, [_vp, ctypes.c_int, _i32, _i32, _i32, _vp, _vp, _vp,
                                            _vp, _vp, _sz, _vp]),
    "sp_expected_recompute": (ctypes.c_int, [_vp, ctypes.c_int, _i32, _i32, _vp, _vp, _i32, _i32,
                                             _i32, _vp, _vp, _vp]),
    "sp_place_checkpoints_frontier": (ctypes.c_int, [_vp, ctypes.c_int, _i32, _i32, _i32, _vp,
                                                     _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "sp_place_checkpoints_grid_workspace_bytes": (_sz, [_i32, _i32, _i32, _i32]),
    "sp_place_checkpoints_grid": (ctypes.c_int, [_vp, ctypes.c_int, _i32, _i32, _i32, _i32, _vp,
                                                 _vp, _vp, _vp, _vp, _sz, _vp]),
    "sp_clip_to_blocks": (ctypes.c_int, [_vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp]),
    "sp_sqrt_positions": (_i32, [_i32, _vp]),
    "sp_log_positions": (_i32, [_i32, _i32, _vp]),
    "sp_balanced_positions": (_i32, [_i32, _i32, _vp]),
    "sp_block_positions": (_i32, [_i32, _i32, _vp]),
    "sp_prefix_index_workspace_bytes": (_sz, [_i32]),
    "sp_prefix_index_build": (ctypes.c_int, [_vp, _vp, _i32, _vp, _vp, _sz, _vp]),
    "sp_match_longest_prefix": (ctypes.c_int, [_vp, _vp, _i32, _vp, _vp, _vp, _i64, _vp, _vp,
                                               _vp]),
    "sp_gamma_observe": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, ctypes.c_double,
                                        _vp]),
    "sp_gamma_snapshot": (ctypes.c_int, [_vp, _vp, _vp, _i32, _i32, ctypes.c_double, _vp, _vp]),
    "sp_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "sp_debug_set": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "sp_debug_get": (ctypes.c_int, [ctypes.c_int]),
    "sp_last_error_string": (ctypes.c_char_p, []),
    "sp_version": (ctypes.c_char_p, []),
}


class SPError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = lib().sp_status_string(status).decode()
        if status == SP_ERR_CUDA:
            msg += " (" + lib().sp_last_error_string().decode() + ")"
        super().__init__(f"{where}: {msg}")


def lib():
    """Load libsparseprefix.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2605_05219_b200.build`"
                               " or __graft_entry__.build() first (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SYMBOLS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(st: int, where: str):
    if st != SP_OK:
        raise SPError(st, where)


def _dev(t: torch.Tensor, dtype, name: str, ndim=None):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be on a CUDA device (no CPU fallback)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if ndim is not None and t.dim() != ndim:
        raise ValueError(f"{name} must be {ndim}-D")
    return t.data_ptr()


def _stream(stream, device):
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def overlap_hist(entry_tokens, entry_off, req_tokens, req_off, req_entry, N, hist=None,
                 lcp_out=None, n_entries=None, stream=None, with_hist=True):
    """a1 + a2.  Returns (hist [E][N+1] int32, accumulated in place; lcp_out [R] or None).
    with_hist=False computes the depths only (lcp_out required)."""
    E = entry_off.numel() - 1 if n_entries is None else n_entries
    R = req_off.numel() - 1
    dev = req_tokens.device
    if hist is None and with_hist:
        hist = torch.zeros(E, N + 1, dtype=torch.int32, device=dev)
    st = lib().sp_overlap_hist(
        _dev(entry_tokens, torch.int32, "entry_tokens"), _dev(entry_off, torch.int64, "entry_off"),
        E, _dev(req_tokens, torch.int32, "req_tokens"), _dev(req_off, torch.int64, "req_off"),
        _dev(req_entry, torch.int32, "req_entry"), R, N,
        _dev(hist, torch.int32, "hist") if with_hist else None,
        None if lcp_out is None else _dev(lcp_out, torch.int32, "lcp_out"), _stream(stream, dev))
    _check(st, "sp_overlap_hist")
    return hist, lcp_out


def accumulate_depths(entry, depth, e_begin, e_end, N, hist, stream=None):
    st = lib().sp_accumulate_depths(_dev(entry, torch.int32, "entry"),
                                    _dev(depth, torch.int32, "depth"), entry.numel(), e_begin,
                                    e_end, N, _dev(hist, torch.int32, "hist"),
                                    _stream(stream, hist.device))
    _check(st, "sp_accumulate_depths")
    return hist


def place_checkpoints_workspace_bytes(n_entries, N, M) -> int:
    return int(lib().sp_place_checkpoints_workspace_bytes(n_entries, N, M))


SP_WS_STATS_BYTES = 256


def dp_stats(workspace) -> dict:
    """Launch statistics from the head of a DP workspace (sp_dp_stats; synchronises)."""
    v = workspace[:64].view(torch.int64).cpu().tolist()
    return {"evaluations": v[0], "entries_i32": v[1], "entries_i64": v[2], "entries_f64": v[3],
            "hull_pops": v[4], "entries_hull": v[5], "hull_event_rows": v[6],
            "entries_hull_big": v[7]}


def place_checkpoints(weights, M, positions=None, n_positions=None, cost=None,
                      cost_by_budget=False, workspace=None, stream=None):
    """a3-a5 (+ a7 for float64 weights).  weights: [E][N+1] int32 / int64 counts or float64.
    Returns (positions [E][M] int32, n_positions [E] int32, cost [E], cost_by_budget or None)."""
    if weights.dim() != 2:
        raise ValueError("weights must be [E][N+1]")
    wtype = _WTYPE.get(weights.dtype)
    if wtype is None:
        raise TypeError("weights must be int32, int64 or float64")
    E, N = weights.shape[0], weights.shape[1] - 1
    dev = weights.device
    cdt = torch.float64 if wtype == SP_W_PROB_F64 else torch.int64
    if positions is None:
        positions = torch.empty(E, max(M, 0), dtype=torch.int32, device=dev)
    if n_positions is None:
        n_positions = torch.empty(E, dtype=torch.int32, device=dev)
    if cost is None:
        cost = torch.empty(E, dtype=cdt, device=dev)
    cbb = None
    if cost_by_budget is True:
        cbb = torch.empty(E, M + 1, dtype=cdt, device=dev)
    elif isinstance(cost_by_budget, torch.Tensor):
        cbb = cost_by_budget
    need = place_checkpoints_workspace_bytes(E, N, M)
    if workspace is None:
        workspace = torch.empty(max(need, 1), dtype=torch.uint8, device=dev)
    st = lib().sp_place_checkpoints(
        _dev(weights, weights.dtype, "weights"), wtype, E, N, M,
        _dev(positions, torch.int32, "positions") if M > 0 else None,
        _dev(n_positions, torch.int32, "n_positions"), _dev(cost, cdt, "cost"),
        None if cbb is None else _dev(cbb, cdt, "cost_by_budget"),
        _dev(workspace, torch.uint8, "workspace"), workspace.numel(), _stream(stream, dev))
    _check(st, "sp_place_checkpoints")
    return positions, n_positions, cost, cbb


def expected_recompute(weights, positions, n_positions, broadcast=True, cost=None, worst=None,
                       stream=None):
    """a6.  broadcast: positions [S][max_pos] / n_positions [S] shared by all entries; else
    [E][S][max_pos] / [E][S].  Returns (cost [E][S], worst [E][S])."""
    wtype = _WTYPE.get(weights.dtype)
    if wtype is None:
        raise TypeError("weights must be int32, int64 or float64")
    E, N = weights.shape[0], weights.shape[1] - 1
    dev = weights.device
    if broadcast:
        S, max_pos = positions.shape[0], positions.shape[1]
    else:
        S, max_pos = positions.shape[1], positions.shape[2]
    cdt = torch.float64 if wtype == SP_W_PROB_F64 else torch.int64
    if cost is None:
        cost = torch.empty(E, S, dtype=cdt, device=dev)
    if worst is None:
        worst = torch.empty(E, S, dtype=torch.int32, device=dev)
    st = lib().sp_expected_recompute(
        _dev(weights, weights.dtype, "weights"), wtype, E, N,
        _dev(positions, torch.int32, "positions") if positions.numel() else None,
        _dev(n_positions, torch.int32, "n_positions"), S, max_pos, 1 if broadcast else 0,
        _dev(cost, cdt, "cost"), _dev(worst, torch.int32, "worst"), _stream(stream, dev))
    _check(st, "sp_expected_recompute")
    return cost, worst


def balanced_positions(N, M):
    buf = (ctypes.c_int32 * max(M, 1))()
    k = lib().sp_balanced_positions(N, M, buf)
    if k < 0:
        raise SPError(-k, "sp_balanced_positions")
    return list(buf[:k])


def block_positions(N, B):
    buf = (ctypes.c_int32 * max(N // max(B, 1), 1))()
    k = lib().sp_block_positions(N, B, buf)
    if k < 0:
        raise SPError(-k, "sp_block_positions")
    return list(buf[:k])


def place_checkpoints_frontier(weights, M, workspace=None, stream=None):
    """f3: positions of every budget m = 1..M from one DP.  Returns (frontier_positions
    [E][M][M] (row m-1 = budget m), frontier_n [E][M], cost_by_budget [E][M+1])."""
    wtype = _WTYPE.get(weights.dtype)
    if wtype is None or weights.dim() != 2:
        raise TypeError("weights must be [E][N+1] int32, int64 or float64")
    E, N = weights.shape[0], weights.shape[1] - 1
    dev = weights.device
    cdt = torch.float64 if wtype == SP_W_PROB_F64 else torch.int64
    fpos = torch.empty(E, M, M, dtype=torch.int32, device=dev)
    fn = torch.empty(E, M, dtype=torch.int32, device=dev)
    cbb = torch.empty(E, M + 1, dtype=cdt, device=dev)
    pos = torch.empty(E, M, dtype=torch.int32, device=dev)
    npos = torch.empty(E, dtype=torch.int32, device=dev)
    cost = torch.empty(E, dtype=cdt, device=dev)
    need = place_checkpoints_workspace_bytes(E, N, M)
    if workspace is None:
        workspace = torch.empty(max(need, 1), dtype=torch.uint8, device=dev)
    st = lib().sp_place_checkpoints_frontier(
        _dev(weights, weights.dtype, "weights"), wtype, E, N, M,
        _dev(fpos, torch.int32, "frontier_positions") if M > 0 else None,
        _dev(fn, torch.int32, "frontier_n") if M > 0 else None, _dev(cbb, cdt, "cbb"),
        _dev(pos, torch.int32, "positions") if M > 0 else None, _dev(npos, torch.int32, "npos"),
        _dev(cost, cdt, "cost"), _dev(workspace, torch.uint8, "workspace"), workspace.numel(),
        _stream(stream, dev))
    _check(st, "sp_place_checkpoints_frontier")
    return fpos, fn, cbb


def place_checkpoints_grid(weights, M, B, positions=None, n_positions=None, cost=None,
                           cost_by_budget=False, workspace=None, stream=None):
    """f1: the exact DP with checkpoints restricted to multiples of B."""
    wtype = _WTYPE.get(weights.dtype)
    if wtype is None or weights.dim() != 2:
        raise TypeError("weights must be [E][N+1] int32, int64 or float64")
    E, N = weights.shape[0], weights.shape[1] - 1
    dev = weights.device
    cdt = torch.float64 if wtype == SP_W_PROB_F64 else torch.int64
    if positions is None:
        positions = torch.empty(E, max(M, 0), dtype=torch.int32, device=dev)
    if n_positions is None:
        n_positions = torch.empty(E, dtype=torch.int32, device=dev)
    if cost is None:
        cost = torch.empty(E, dtype=cdt, device=dev)
    cbb = torch.empty(E, M + 1, dtype=cdt, device=dev) if cost_by_budget is True else (
        cost_by_budget if isinstance(cost_by_budget, torch.Tensor) else None)
    need = int(lib().sp_place_checkpoints_grid_workspace_bytes(E, N, M, B))
    if workspace is None:
        workspace = torch.empty(max(need, 1), dtype=torch.uint8, device=dev)
    st = lib().sp_place_checkpoints_grid(
        _dev(weights, weights.dtype, "weights"), wtype, E, N, M, B,
        _dev(positions, torch.int32, "positions") if M > 0 else None,
        _dev(n_positions, torch.int32, "n_positions"), _dev(cost, cdt, "cost"),
        None if cbb is None else _dev(cbb, cdt, "cost_by_budget"),
        _dev(workspace, torch.uint8, "workspace"), workspace.numel(), _stream(stream, dev))
    _check(st, "sp_place_checkpoints_grid")
    return positions, n_positions, cost, cbb


def clip_to_blocks(positions, n_positions, B, out=None, out_n=None, stream=None):
    """f1: floor every position to a multiple of B, drop zeros, merge duplicates."""
    E, max_pos = positions.shape
    dev = positions.device
    out = torch.empty_like(positions) if out is None else out
    out_n = torch.empty_like(n_positions) if out_n is None else out_n
    st = lib().sp_clip_to_blocks(_dev(positions, torch.int32, "positions") if max_pos else None,
                                 _dev(n_positions, torch.int32, "n_positions"), E, max_pos, B,
                                 _dev(out, torch.int32, "out") if max_pos else None,
                                 _dev(out_n, torch.int32, "out_n"), _stream(stream, dev))
    _check(st, "sp_clip_to_blocks")
    return out, out_n


def sqrt_positions(N):
    buf = (ctypes.c_int32 * max(N, 1))()
    k = lib().sp_sqrt_positions(N, buf)
    if k < 0:
        raise SPError(-k, "sp_sqrt_positions")
    return list(buf[:k])


def log_positions(N, M):
    buf = (ctypes.c_int32 * max(M, 1))()
    k = lib().sp_log_positions(N, M, buf)
    if k < 0:
        raise SPError(-k, "sp_log_positions")
    return list(buf[:k])


def baseline_sets(N, budgets=(), blocks=(), device="cuda"):
    """Pack balanced schedules (one per budget) and block schedules (one per B) as broadcast
    placement sets for expected_recompute: returns (positions [S][max_pos], n_positions [S],
    labels)."""
    sets, labels = [], []
    for m in budgets:
        sets.append(balanced_positions(N, m))
        labels.append(("balanced", m))
    for B in blocks:
        sets.append(block_positions(N, B))
        labels.append(("block", B))
    width = max([len(s) for s in sets] + [1])
    pos = torch.zeros(len(sets), width, dtype=torch.int32)
    for i, s in enumerate(sets):
        if s:
            pos[i, :len(s)] = torch.tensor(s, dtype=torch.int32)
    npos = torch.tensor([len(s) for s in sets], dtype=torch.int32)
    return pos.to(device), npos.to(device), labels


# ---------------------------------------------------------------------------------------------
# f2: Thm 4's exponentially weighted histogram
# ---------------------------------------------------------------------------------------------
class GammaEstimator:
    """Device state of E per-entry estimators (W [E][N+1] f64, t [E], tau [E] int64)."""

    def __init__(self, n_entries, N, gamma=0.99, device="cuda"):
        self.N, self.gamma = N, float(gamma)
        self.W = torch.zeros(n_entries, N + 1, dtype=torch.float64, device=device)
        self.t = torch.zeros(n_entries, dtype=torch.int64, device=device)
        self.tau = torch.zeros(n_entries, dtype=torch.int64, device=device)

    def observe(self, obs_off, depth, stream=None):
        """Append one batch: obs_off int64 [E+1] CSR offsets, depth int32 (grouped by entry,
        arrival order within an entry)."""
        gamma_observe(self.W, self.t, self.tau, obs_off, depth, self.gamma, stream)

    def snapshot(self, out=None, stream=None):
        return gamma_snapshot(self.W, self.t, self.tau, self.gamma, out, stream)


def gamma_observe(W, t, tau, obs_off, depth, gamma, stream=None):
    E, N = W.shape[0], W.shape[1] - 1
    st = lib().sp_gamma_observe(_dev(W, torch.float64, "W"), _dev(t, torch.int64, "t"),
                                _dev(tau, torch.int64, "tau"), _dev(obs_off, torch.int64, "obs_off"),
                                _dev(depth, torch.int32, "depth"), E, N, float(gamma),
                                _stream(stream, W.device))
    _check(st, "sp_gamma_observe")


def gamma_snapshot(W, t, tau, gamma, out=None, stream=None):
    E, N = W.shape[0], W.shape[1] - 1
    if out is None:
        out = torch.empty_like(W)
    st = lib().sp_gamma_snapshot(_dev(W, torch.float64, "W"), _dev(t, torch.int64, "t"),
                                 _dev(tau, torch.int64, "tau"), E, N, float(gamma),
                                 _dev(out, torch.float64, "p_out"), _stream(stream, W.device))
    _check(st, "sp_gamma_snapshot")
    return out


# ---------------------------------------------------------------------------------------------
# f4: longest-prefix search over all cached entries
# ---------------------------------------------------------------------------------------------
class PrefixIndex:
    """Sorted-token index of a set of cached entries (device).  Rebuild when the cache changes."""

    def __init__(self, entry_tokens, entry_off, insertion=None, stream=None):
        self.entry_tokens, self.entry_off = entry_tokens, entry_off
        self.E = entry_off.numel() - 1
        dev = entry_off.device
        nb = int(lib().sp_prefix_index_workspace_bytes(self.E))
        self.ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=dev)
        ins = None if insertion is None else _dev(insertion, torch.int64, "insertion")
        tok = _dev(entry_tokens, torch.int32, "entry_tokens") if entry_tokens.numel() else None
        st = lib().sp_prefix_index_build(tok, _dev(entry_off, torch.int64, "entry_off"), self.E,
                                         ins, _dev(self.ws, torch.uint8, "index"), nb,
                                         _stream(stream, dev))
        _check(st, "sp_prefix_index_build")

    def match(self, req_tokens, req_off, out_entry=None, out_depth=None, stream=None):
        """Returns (match_entry [R] int32, -1 = none; match_depth [R] int32, the raw LCP)."""
        R = req_off.numel() - 1
        dev = req_off.device
        if out_entry is None:
            out_entry = torch.empty(max(R, 0), dtype=torch.int32, device=dev)
        if out_depth is None:
            out_depth = torch.empty(max(R, 0), dtype=torch.int32, device=dev)
        if R == 0:
            return out_entry, out_depth
        tok = _dev(self.entry_tokens, torch.int32, "entry_tokens") if self.entry_tokens.numel() else None
        st = lib().sp_match_longest_prefix(
            tok, _dev(self.entry_off, torch.int64, "entry_off"), self.E,
            _dev(self.ws, torch.uint8, "index"),
            _dev(req_tokens, torch.int32, "req_tokens") if req_tokens.numel() else None,
            _dev(req_off, torch.int64, "req_off"), R, _dev(out_entry, torch.int32, "match_entry"),
            _dev(out_depth, torch.int32, "match_depth"), _stream(stream, dev))
        _check(st, "sp_match_longest_prefix")
        return out_entry, out_depth


# ---------------------------------------------------------------------------------------------
# comparison / test hooks
# ---------------------------------------------------------------------------------------------
class debug:
    """Context manager: `with sp.debug(SP_DBG_NO_HULL=1): ...` sets process-wide kernel-path
    hooks (sp_debug_set) and restores the previous values on exit."""

    def __init__(self, **flags):
        self.flags = {globals()[k]: int(v) for k, v in flags.items()}
        self.prev = {}

    def __enter__(self):
        for f, v in self.flags.items():
            self.prev[f] = int(lib().sp_debug_set(f, v))
        return self

    def __exit__(self, *exc):
        for f, v in self.prev.items():
            lib().sp_debug_set(f, v)
        return False
