"""Seeded synthetic workloads (W1-W5) -- inputs only.

This module is the ONE piece shared by the oracle side (tests, CPU baseline) and the CUDA side.
It holds none of the method's arithmetic: it draws overlap depths from the shape laws of
Fig. 1 (shapes as in S:70-78) and materialises token traces whose LCP equals the
drawn depth by construction (fresh suffix tokens come from an id range disjoint from the entry
tokens).  Dense "depth-mode" histograms are drawn the same way.

Everything is counter-based (a 32-bit integer hash of (seed, stream, index)), written with
plain torch integer ops so that the same code runs on CPU (tests) and on the GPU (bench inputs,
tens of GB).  No value produced here ever comes from the CUDA path.

Recipe:
  entry tokens         uniform in [0, 2^18)
  request suffix ids   uniform in [2^20, 2^21)   (disjoint => LCP(request, entry) = depth)
  depth laws, on [1, L] with L the entry length:
    uniform      U[1, L]
    end_spike    0.9: U[L-63, L]; 0.1: U[1, L]                       (QuALITY-like)
    head_heavy   0.8: 1 + Geometric(mean 32) capped at L; 0.2: U[1,L] (System Prompts)
    multimodal   3 truncated discrete Gaussians, sigma = L/24        (NarrativeQA-like)
    mix          entry e uses shape (uniform, end_spike, head_heavy, multimodal)[e % 4]
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

MASK32 = 0xFFFFFFFF
ENTRY_VOCAB = 1 << 18
SUFFIX_BASE = 1 << 20
SUFFIX_VOCAB = 1 << 20
SHAPES = ("uniform", "end_spike", "head_heavy", "multimodal")

# ---------------------------------------------------------------------------------------------
# counter-based hashing (lowbias32 finaliser); products are split so nothing overflows int64
# ---------------------------------------------------------------------------------------------


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    lo = (x & 0xFFFF) * c
    hi = (((x >> 16) & 0xFFFF) * c) & 0xFFFF
    return (lo + (hi << 16)) & MASK32


def hash32(x: torch.Tensor) -> torch.Tensor:
    x = x & MASK32
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def stream(seed: int, *keys) -> torch.Tensor:
    """hash of (seed, k1, k2, ...) where each key is an int or an int64 tensor."""
    h = None
    dev = next((k.device for k in keys if isinstance(k, torch.Tensor)), torch.device("cpu"))
    h = hash32(torch.tensor(seed & MASK32, dtype=torch.int64, device=dev))
    for k in keys:
        if not isinstance(k, torch.Tensor):
            k = torch.tensor(int(k) & MASK32, dtype=torch.int64, device=dev)
        h = hash32(h ^ (k & MASK32))
    return h


def uniform01(seed: int, *keys) -> torch.Tensor:
    return stream(seed, *keys).to(torch.float64) * (1.0 / 4294967296.0)


def randint(seed: int, lo, hi, *keys) -> torch.Tensor:
    """integers in [lo, hi] (inclusive); lo/hi may be tensors."""
    u = uniform01(seed, *keys)
    span = (hi - lo + 1)
    if isinstance(span, torch.Tensor):
        span = span.to(torch.float64)
    v = torch.floor(u * span).to(torch.int64)
    return lo + v


# ---------------------------------------------------------------------------------------------
# depth laws (Fig. 1 shapes); L: int64 tensor of entry lengths per sample
# ---------------------------------------------------------------------------------------------


def draw_depths(shape: torch.Tensor, L: torch.Tensor, seed: int, ent: torch.Tensor,
                idx: torch.Tensor) -> torch.Tensor:
    """shape: int64 shape id per sample (index into SHAPES); returns depths in [1, L]."""
    Lf = L.to(torch.float64)
    u1 = uniform01(seed, 1, ent, idx)
    u2 = uniform01(seed, 2, ent, idx)
    u3 = uniform01(seed, 3, ent, idx)
    uni = 1 + torch.floor(u2 * Lf).to(torch.int64)
    # end_spike: 0.9 of the mass on the last 64 positions
    spike = L - 63 + torch.floor(u2 * 64.0).to(torch.int64)
    end_spike = torch.where(u1 < 0.9, spike, uni)
    # head_heavy: 0.8 geometric with mean 32 from depth 1
    geo = 1 + torch.floor(torch.log1p(-u2) / math.log(1.0 - 1.0 / 32.0)).to(torch.int64)
    head = torch.where(u1 < 0.8, geo, uni)
    # multimodal: 3 modes per entry, centres drawn per entry, sigma = L/24
    mode = torch.floor(u1 * 3.0).to(torch.int64)
    centre = 1.0 + uniform01(seed, 4, ent, mode) * (Lf - 1.0)
    z = torch.sqrt(-2.0 * torch.log1p(-u2)) * torch.cos(2.0 * math.pi * u3)
    multi = torch.round(centre + z * (Lf / 24.0)).to(torch.int64)
    d = torch.where(shape == 0, uni,
                    torch.where(shape == 1, end_spike, torch.where(shape == 2, head, multi)))
    return torch.minimum(torch.maximum(d, torch.ones_like(d)), L)


def shape_ids(name: str, ent: torch.Tensor) -> torch.Tensor:
    if name == "mix":
        return ent % 4
    return torch.full_like(ent, SHAPES.index(name))


# ---------------------------------------------------------------------------------------------
# configurations (SURVEY 8(d) W1-W5 = BASELINE.json "configs")
# ---------------------------------------------------------------------------------------------


@dataclass(frozen=True)
class TraceConfig:
    name: str
    n_entries: int
    N: int
    M: int
    req_per_entry: int
    L_range: tuple          # entry length range (inclusive)
    suffix_range: tuple     # fresh-suffix length range (inclusive)
    shape: str              # depth law of the LCP trace
    miss_frac: float = 0.0  # fraction of requests with depth 0 (a miss, bin 0)
    align: int = 4          # pad lengths so every CSR offset is a multiple of `align` tokens
    dense_n: tuple = None   # (lo, hi) draws per entry for the dense DP histogram, or None
    dense_shape: str = "mix"
    M_sweep: tuple = field(default=())


CONFIGS = {
    "W1": TraceConfig("W1", 1, 64, 4, 100, (64, 64), (1, 8), "multimodal", align=1),
    "W2": TraceConfig("W2", 1000, 2048, 8, 64, (1024, 2048), (32, 512), "head_heavy"),
    "W3": TraceConfig("W3", 2000, 8192, 16, 20, (5000, 8000), (16, 128), "end_spike"),
    "W4": TraceConfig("W4", 2000, 8192, 64, 20, (5000, 8192), (16, 128), "end_spike",
                      dense_n=(4096, 4096), M_sweep=tuple(range(1, 65))),
    "W5": TraceConfig("W5", 16384, 32768, 64, 20, (24576, 32768), (16, 128), "end_spike",
                      dense_n=(8192, 16384)),
}


def scaled(cfg: TraceConfig, n_entries: int) -> TraceConfig:
    """Same shapes and sizes per entry, fewer entries (parity-test cases)."""
    d = dict(cfg.__dict__)
    d["n_entries"] = n_entries
    d["name"] = f"{cfg.name}[E={n_entries}]"
    return TraceConfig(**d)


# ---------------------------------------------------------------------------------------------
# token traces
# ---------------------------------------------------------------------------------------------


def _round_up(x: torch.Tensor, a: int) -> torch.Tensor:
    return (x + (a - 1)) // a * a if a > 1 else x


def make_trace(cfg: TraceConfig, seed: int = 0, device="cpu", entry_begin: int = 0,
               n_req_entries: int = None, chunk: int = 1 << 27, world: int = 1,
               rank: int = 0) -> dict:
    """Entry token CSR + request token CSR for cfg.

    Requests are generated for entries [entry_begin, entry_begin + n_req_entries) (all entries
    by default); with world > 1 only the requests that "arrive" at `rank` are materialised
    (request g arrives at rank hash(g) % world: uniformly at random).  Returns a
    dict of tensors on `device`: entry_tokens int32, entry_off int64 [E+1], req_tokens int32,
    req_off int64 [R+1], req_entry int32 [R], depth int32 [R] (the drawn depth = the LCP by
    construction, not clamped to N), N (int).
    """
    dev = torch.device(device)
    E, a = cfg.n_entries, max(cfg.align, 1)
    ent = torch.arange(E, dtype=torch.int64, device=dev)
    L = randint(seed, cfg.L_range[0], cfg.L_range[1], 10, ent)
    if a > 1:
        L = torch.clamp(L // a * a, min=a)
    L = torch.clamp(L, max=cfg.N)
    entry_off = torch.zeros(E + 1, dtype=torch.int64, device=dev)
    entry_off[1:] = torch.cumsum(L, 0)
    n_tok = int(entry_off[-1])
    entry_tokens = torch.empty(n_tok, dtype=torch.int32, device=dev)
    for p0 in range(0, n_tok, chunk):
        p = torch.arange(p0, min(p0 + chunk, n_tok), dtype=torch.int64, device=dev)
        entry_tokens[p0:p0 + p.numel()] = (stream(seed, 11, p) & (ENTRY_VOCAB - 1)).to(torch.int32)

    nre = E - entry_begin if n_req_entries is None else n_req_entries
    re = torch.arange(entry_begin, entry_begin + nre, dtype=torch.int64, device=dev)
    req_entry = re.repeat_interleave(cfg.req_per_entry)
    ridx = torch.arange(cfg.req_per_entry, dtype=torch.int64, device=dev).repeat(nre)
    gid = req_entry * cfg.req_per_entry + ridx          # global request id (rank independent)
    if world > 1:
        mine = (stream(seed, 15, gid) % world) == rank
        req_entry, ridx, gid = req_entry[mine], ridx[mine], gid[mine]
    Lr = L[req_entry]
    depth = draw_depths(shape_ids(cfg.shape, req_entry), Lr, seed, req_entry, ridx)
    if cfg.miss_frac > 0:
        miss = uniform01(seed, 12, gid) < cfg.miss_frac
        depth = torch.where(miss, torch.zeros_like(depth), depth)
    suf = randint(seed, cfg.suffix_range[0], cfg.suffix_range[1], 13, gid)
    rlen = _round_up(depth + suf, a)
    req_off = torch.zeros(rlen.numel() + 1, dtype=torch.int64, device=dev)
    req_off[1:] = torch.cumsum(rlen, 0)
    n_rt = int(req_off[-1])
    req_tokens = torch.empty(n_rt, dtype=torch.int32, device=dev)
    for p0 in range(0, n_rt, chunk):
        p = torch.arange(p0, min(p0 + chunk, n_rt), dtype=torch.int64, device=dev)
        r = torch.searchsorted(req_off, p, right=True) - 1
        k = p - req_off[r]
        e = req_entry[r]
        from_entry = k < depth[r]
        src = torch.where(from_entry, entry_off[e] + k, torch.zeros_like(k))
        suffix = SUFFIX_BASE + (stream(seed, 14, gid[r], k) & (SUFFIX_VOCAB - 1))
        tok = torch.where(from_entry, entry_tokens[src].to(torch.int64), suffix)
        req_tokens[p0:p0 + p.numel()] = tok.to(torch.int32)
    return dict(entry_tokens=entry_tokens, entry_off=entry_off, req_tokens=req_tokens,
                req_off=req_off, req_entry=req_entry.to(torch.int32),
                depth=depth.to(torch.int32), N=cfg.N, L=L)


def make_dense_hist(cfg: TraceConfig, seed: int = 0, device="cpu", entry_begin: int = 0,
                    n_entries: int = None, chunk: int = 1 << 26) -> torch.Tensor:
    """Depth-mode histograms: n_e ~ U[dense_n] draws per entry from the entry's law on
    [1, L_e], L_e ~ U[3N/4, N].  Returns int32 [E][N+1] counts (bin 0 = 0)."""
    dev = torch.device(device)
    lo, hi = cfg.dense_n
    E = cfg.n_entries - entry_begin if n_entries is None else n_entries
    N = cfg.N
    ent = torch.arange(entry_begin, entry_begin + E, dtype=torch.int64, device=dev)
    n = randint(seed, lo, hi, 20, ent)
    L = randint(seed, (3 * N) // 4, N, 21, ent)
    hist = torch.zeros(E * (N + 1), dtype=torch.int32, device=dev)
    # process entries in groups so the per-draw temporaries stay bounded
    per = max(1, chunk // max(hi, 1))
    for g0 in range(0, E, per):
        g1 = min(E, g0 + per)
        ng = n[g0:g1]
        le = torch.arange(g0, g1, dtype=torch.int64, device=dev).repeat_interleave(ng)
        start = torch.zeros(g1 - g0, dtype=torch.int64, device=dev)
        start[1:] = torch.cumsum(ng, 0)[:-1]
        idx = torch.arange(le.numel(), dtype=torch.int64, device=dev) - start[le - g0]
        ge = ent[le]
        d = draw_depths(shape_ids(cfg.dense_shape, ge), L[le], seed + 7919, ge, idx)
        flat = le * (N + 1) + d
        hist.index_add_(0, flat, torch.ones_like(flat, dtype=torch.int32))
    return hist.view(E, N + 1)


def uniform_hist(n_entries: int, N: int, device="cpu") -> torch.Tensor:
    """All-ones histograms (c_t = 1 for t = 1..N): the Thm 1 case."""
    h = torch.ones(n_entries, N + 1, dtype=torch.int32, device=device)
    h[:, 0] = 0
    return h


def random_small_hist(seed: int, N: int, max_count: int = 5, zero_frac: float = 0.3,
                      key: int = 0) -> torch.Tensor:
    """Small random histograms for exhaustive tests: c_t in [0, max_count], ~zero_frac zeros."""
    t = torch.arange(N + 1, dtype=torch.int64)
    c = randint(seed, 0, max_count, 30, key, t)
    z = uniform01(seed, 31, key, t) < zero_frac
    c = torch.where(z, torch.zeros_like(c), c)
    c[0] = 0
    return c
