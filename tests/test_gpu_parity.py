"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit-exact for every
integer output (positions, counts, int64 costs, LCPs, histograms); fp64 variant within 1e-12
relative error of the exact rational reference V_int / n (BASELINE.json north_star)."""
import os

import numpy as np
import pytest
import torch

import oracle
from _bounds import f64_within
from paper_2605_05219_b200 import sp
from paper_2605_05219_b200 import workload as wl

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2605_05219_b200 import build
    build.build()
    sp.lib()
    return torch.device("cuda:0")


def np_(t):
    return t.detach().cpu().numpy()


def run_lcp(tr, N, dev, E):
    g = {k: v.to(dev) for k, v in tr.items() if isinstance(v, torch.Tensor)}
    R = g["req_off"].numel() - 1
    lcp = torch.full((R,), -7, dtype=torch.int32, device=dev)
    hist, _ = sp.overlap_hist(g["entry_tokens"], g["entry_off"], g["req_tokens"], g["req_off"],
                              g["req_entry"], N, lcp_out=lcp, n_entries=E)
    torch.cuda.synchronize()
    return np_(hist), np_(lcp)


def oracle_lcp(tr, N, E):
    return oracle.lcp_hist(np_(tr["entry_tokens"]), np_(tr["entry_off"]), np_(tr["req_tokens"]),
                           np_(tr["req_off"]), np_(tr["req_entry"]), N, n_entries=E, nthreads=8)


# ------------------------------------------------------------------------------------------
# a1 + a2 : LCP + histogram
# ------------------------------------------------------------------------------------------


@pytest.mark.parametrize("name,E,align", [("W1", 1, 1), ("W2", 40, 4), ("W2", 40, 1),
                                          ("W3", 12, 4), ("W3", 12, 1)])
def test_lcp_hist_parity(dev, name, E, align):
    cfg = wl.scaled(wl.CONFIGS[name], E)
    cfg = wl.TraceConfig(**{**cfg.__dict__, "align": align, "miss_frac": 0.05})
    tr = wl.make_trace(cfg, seed=3)
    h_gpu, l_gpu = run_lcp(tr, cfg.N, dev, E)
    h_ref, l_ref = oracle_lcp(tr, cfg.N, E)
    assert (l_gpu == l_ref).all()
    assert (h_gpu == h_ref).all()
    # and the construction: LCP = drawn depth (clamped to N)
    assert (l_gpu == np.minimum(np_(tr["depth"]), cfg.N)).all()


def test_lcp_clamp_ragged_and_bad_entries(dev):
    """N smaller than the overlaps (clamp), empty requests, out-of-range entry ids, and an
    accumulate (+=) into a non-zero histogram."""
    cfg = wl.scaled(wl.CONFIGS["W2"], 9)
    tr = wl.make_trace(cfg, seed=4)
    N = 300
    tr["req_entry"][5] = 99          # out of range -> skipped, lcp = -1
    tr["req_entry"][6] = -1
    # make request 7 empty
    off = tr["req_off"].clone()
    L7 = int(off[8] - off[7])
    keep = torch.ones(tr["req_tokens"].numel(), dtype=torch.bool)
    keep[int(off[7]):int(off[8])] = False
    tr["req_tokens"] = tr["req_tokens"][keep]
    off[8:] -= L7
    tr["req_off"] = off
    g = {k: v.to(dev) for k, v in tr.items() if isinstance(v, torch.Tensor)}
    R = off.numel() - 1
    base = torch.randint(0, 5, (9, N + 1), dtype=torch.int32)
    hist = base.clone().to(dev)
    lcp = torch.zeros(R, dtype=torch.int32, device=dev)
    sp.overlap_hist(g["entry_tokens"], g["entry_off"], g["req_tokens"], g["req_off"],
                    g["req_entry"], N, hist=hist, lcp_out=lcp, n_entries=9)
    torch.cuda.synchronize()
    # the oracle rejects bad entry ids as an error: give those requests entry 0 there and
    # remove their contribution afterwards
    valid = np.ones(R, bool)
    valid[[5, 6]] = False
    ok_entry = np_(tr["req_entry"]).copy()
    ok_entry[~valid] = 0
    ref_h, ref_l = oracle.lcp_hist(np_(tr["entry_tokens"]), np_(tr["entry_off"]),
                                   np_(tr["req_tokens"]), np_(off), ok_entry, N, n_entries=9)
    got_l = np_(lcp)
    assert (got_l[valid] == ref_l[valid]).all()
    assert (got_l[~valid] == -1).all()
    assert got_l[7] == 0
    # remove the two substituted requests from the oracle histogram
    for r in (5, 6):
        ref_h[0, ref_l[r]] -= 1
    assert (np_(hist) == np_(base) + ref_h).all()


def test_lcp_w5_full_size_sampled(dev):
    """BASELINE's scale config at full size (16384 entries x N=32768, 20 requests each, ~36 GB of
    request tokens) in the bench's launch configuration: sampled requests' LCPs and sampled
    entries' whole histogram rows against the oracle's literal LCP loop, one by one; the
    drawn depth (the LCP by construction) for every request."""
    cfg = wl.CONFIGS["W5"]
    tr = wl.make_trace(cfg, seed=0, device=dev)
    E, N = cfg.n_entries, cfg.N
    R = tr["req_off"].numel() - 1
    lcp = torch.full((R,), -7, dtype=torch.int32, device=dev)
    hist, _ = sp.overlap_hist(tr["entry_tokens"], tr["entry_off"], tr["req_tokens"], tr["req_off"],
                              tr["req_entry"], N, lcp_out=lcp, n_entries=E)
    torch.cuda.synchronize()
    assert torch.equal(lcp, torch.clamp(tr["depth"], max=N))
    eo, ro, re_ = np_(tr["entry_off"]), np_(tr["req_off"]), np_(tr["req_entry"])
    lcp_h = np_(lcp)

    def one_entry(e, reqs):
        et = np_(tr["entry_tokens"][int(eo[e]):int(eo[e + 1])])
        rts = [np_(tr["req_tokens"][int(ro[r]):int(ro[r + 1])]) for r in reqs]
        roff = np.concatenate([[0], np.cumsum([len(x) for x in rts])]).astype(np.int64)
        rtok = np.concatenate(rts).astype(np.int32) if rts else np.zeros(0, np.int32)
        return oracle.lcp_hist(et, np.array([0, len(et)], np.int64), rtok, roff,
                               np.zeros(len(reqs), np.int32), N, n_entries=1)

    rng = np.random.default_rng(0)
    for r in rng.choice(R, 64, replace=False):       # sampled requests
        _, rl = one_entry(int(re_[r]), [int(r)])
        assert lcp_h[r] == rl[0], r
    for e in (0, 1, 4097, 16383):                     # sampled entries: their whole rows
        reqs = np.nonzero(re_ == e)[0]
        rh, _ = one_entry(e, [int(r) for r in reqs])
        assert (np_(hist[e]) == rh[0]).all(), e


def test_expected_recompute_w5_full_size_sampled(dev):
    """The bench's a6 call at full W5 size (16384 dense rows, the balanced-64 and block-64/128
    sets, broadcast): sampled entries against the oracle's definitional evaluation; worst cases
    against the closed forms at every entry."""
    cfg = wl.CONFIGS["W5"]
    H = wl.make_dense_hist(cfg, seed=0, device=dev)
    pos, npos, labels = sp.baseline_sets(cfg.N, budgets=(cfg.M,), blocks=(64, 128), device=dev)
    cost, worst = sp.expected_recompute(H, pos, npos, broadcast=True)
    torch.cuda.synchronize()
    rows = [0, 1, 2, 777, 4097, 8191, 12000, 16383]
    rc, rw = oracle.eval_batch(np_(H[rows]), np_(pos), np_(npos), broadcast=True, nthreads=8)
    assert (np_(cost)[rows] == rc).all() and (np_(worst)[rows] == rw).all()
    N = cfg.N
    assert (np_(worst)[:, 0] == -(-(N + 1) // (cfg.M + 1)) - 1).all()   # Thm 1.2 tail
    assert (np_(worst)[:, 1] == 63).all() and (np_(worst)[:, 2] == 127).all()   # block B: B - 1
    assert (np_(cost) >= 0).all()


def test_accumulate_depths(dev):
    rng = np.random.default_rng(5)
    n, E, N = 20000, 50, 700
    ent = rng.integers(-3, E + 3, n).astype(np.int32)
    dep = rng.integers(-2, N + 3, n).astype(np.int32)
    hist = torch.zeros(20, N + 1, dtype=torch.int32, device=dev)
    sp.accumulate_depths(torch.from_numpy(ent).to(dev), torch.from_numpy(dep).to(dev), 10, 30, N,
                         hist)
    ref = np.zeros((20, N + 1), np.int64)
    m = (ent >= 10) & (ent < 30) & (dep >= 0) & (dep <= N)
    np.add.at(ref, (ent[m] - 10, dep[m]), 1)
    assert (np_(hist) == ref).all()


# ------------------------------------------------------------------------------------------
# a3 - a5 : the DP
# ------------------------------------------------------------------------------------------


def gpu_place(H, M, dev, dtype=torch.int32):
    w = torch.as_tensor(H).to(dtype).to(dev).contiguous()
    pos, npos, cost, cbb = sp.place_checkpoints(w, M, cost_by_budget=True)
    torch.cuda.synchronize()
    return np_(pos), np_(npos), np_(cost), np_(cbb)


def check_against_oracle(H, M, pos, npos, cost, cbb, algo="cht", rows=None):
    rows = range(H.shape[0]) if rows is None else rows
    for e in rows:
        c = H[e].astype(np.int64)
        rp, rc, rcbb = oracle.place(c, M, algo)
        k = len(rp)
        assert npos[e] == k, (e, npos[e], k)
        assert pos[e, :k].tolist() == rp.tolist(), (e, pos[e, :k], rp)
        assert (pos[e, k:] == 0).all()
        assert cost[e] == rc, (e, cost[e], rc)
        assert (cbb[e] == rcbb).all(), e


def test_dp_small_exhaustive(dev):
    """Every N <= 16, every M <= N, random sparse/dense histograms: GPU == naive oracle."""
    for N in range(1, 17):
        H = np.stack([wl.random_small_hist(21, N, max_count=6, zero_frac=z, key=k).numpy()
                      for k, z in enumerate([0.0, 0.3, 0.6, 0.9] * 6)])
        for M in range(0, N + 1):
            pos, npos, cost, cbb = gpu_place(H, M, dev)
            check_against_oracle(H, M, pos, npos, cost, cbb, algo="naive")


def test_dp_w1(dev):
    cfg = wl.CONFIGS["W1"]
    tr = wl.make_trace(cfg, seed=0)
    h, _ = oracle_lcp(tr, cfg.N, 1)
    pos, npos, cost, cbb = gpu_place(h, cfg.M, dev)
    bpos, bcost = oracle.brute_force(h[0].astype(np.int64), cfg.M)
    assert cost[0] == bcost and pos[0, :npos[0]].tolist() == bpos.tolist()
    check_against_oracle(h, cfg.M, pos, npos, cost, cbb, algo="naive")


@pytest.mark.parametrize("N,M,E", [(97, 5, 33), (300, 20, 20), (1000, 8, 12), (2048, 8, 40),
                                   (4097, 16, 10)])
def test_dp_dense_random(dev, N, M, E):
    cfg = wl.TraceConfig("t", E, N, M, 1, (N, N), (1, 1), "uniform", dense_n=(N // 2, 4 * N))
    H = wl.make_dense_hist(cfg, seed=N).numpy()
    pos, npos, cost, cbb = gpu_place(H, M, dev)
    check_against_oracle(H, M, pos, npos, cost, cbb, algo="naive" if N <= 1000 else "cht")


@pytest.mark.parametrize("name", ["W2", "W3"])
def test_dp_from_lcp_traces(dev, name):
    """W2/W3-shaped histograms from LCP traces (sparse: K <= requests/entry).  The input comes
    from the oracle's LCP loop, never from the CUDA path."""
    cfg = wl.scaled(wl.CONFIGS[name], 24)
    tr = wl.make_trace(cfg, seed=6)
    h, _ = oracle_lcp(tr, cfg.N, 24)
    pos, npos, cost, cbb = gpu_place(h, cfg.M, dev)
    check_against_oracle(h, cfg.M, pos, npos, cost, cbb)


def test_dp_w4_budget_sweep_sample(dev):
    cfg = wl.scaled(wl.CONFIGS["W4"], 64)
    H = wl.make_dense_hist(cfg, seed=2).numpy()
    pos, npos, cost, cbb = gpu_place(H, 64, dev)
    check_against_oracle(H, 64, pos, npos, cost, cbb, rows=range(0, 64, 7))


def thm1_value(N, M):
    K = M + 1
    q, rho = divmod(N + 1, K)
    return (K - rho) * q * (q - 1) // 2 + rho * q * (q + 1) // 2


def test_dp_uniform_thm1_full_size(dev):
    """Thm 1 closed form and the F7 positions at W5's N, M (no oracle needed)."""
    N, M = 32768, 64
    H = wl.uniform_hist(8, N).numpy()
    pos, npos, cost, cbb = gpu_place(H, M, dev)
    K = M + 1
    q, rho = divmod(N + 1, K)
    f7 = [i * q + max(0, i - (K - rho)) for i in range(1, M + 1)]
    for e in range(8):
        assert cost[e] == thm1_value(N, M)
        assert [int(x) for x in cbb[e]] == [thm1_value(N, m) for m in range(M + 1)]
        assert npos[e] == M and pos[e].tolist() == f7


def test_dp_uniform_thm1_bench_size(dev):
    """The bench's all-ones variant (`--dp-hist ones`, 16384 x N=32768 x M=64, the one-warp
    kernel's hand-off to the large-hull mode): every entry's V_0..V_M equal Thm 1's closed form
     and its positions SURVEY F7's rule-B formula; no entry on the D&C kernel."""
    N, M, E = 32768, 64, 16384
    H = wl.uniform_hist(E, N, device=dev)
    ws = torch.empty(sp.place_checkpoints_workspace_bytes(E, N, M), dtype=torch.uint8, device=dev)
    pos, npos, cost, cbb = sp.place_checkpoints(H, M, cost_by_budget=True, workspace=ws)
    torch.cuda.synchronize()
    st = sp.dp_stats(ws)
    assert st["entries_hull"] == E and st["entries_hull_big"] == E and st["evaluations"] == 0
    K = M + 1
    q, rho = divmod(N + 1, K)
    f7 = torch.tensor([i * q + max(0, i - (K - rho)) for i in range(1, M + 1)], dtype=torch.int32,
                      device=dev)
    v = torch.tensor([thm1_value(N, m) for m in range(M + 1)], dtype=torch.int64, device=dev)
    assert bool((npos == M).all()) and bool((pos == f7).all())
    assert bool((cost == thm1_value(N, M)).all()) and bool((cbb == v).all())


def test_dp_w5_full_size_every_entry(dev):
    """BASELINE's scale config at full size (16384 x N=32768 x M=64) in the bench launch
    configuration; EVERY entry against the oracle's CHT DP (threaded over the host
    cores): positions, counts, V_M and V_0..V_M bit-exact."""
    cfg = wl.CONFIGS["W5"]
    H = wl.make_dense_hist(cfg, seed=0, device=dev)
    pos, npos, cost, cbb = sp.place_checkpoints(H, cfg.M, cost_by_budget=True)
    torch.cuda.synchronize()
    pos, npos, cost, cbb = np_(pos), np_(npos), np_(cost), np_(cbb)
    Hc = np_(H)
    del H
    rpos, rnpos, rcost, rcbb = oracle.place_batch(Hc, cfg.M, "cht", nthreads=os.cpu_count() or 1,
                                                  with_budget=True)
    assert (npos == rnpos).all()
    assert (pos == rpos).all()
    assert (cost == rcost).all()
    assert (cbb == rcbb).all()
    assert (npos == cfg.M).all()                      # dense histograms: every slot is used


def test_dp_accum_full_size_every_entry(dev):
    """The bench's `--dp-hist accum` variant at full size (16384 x N=32768 x M=64, n ~ U[1.2e5,
    1.8e5] per row: past the int32 guard, so the int32 kernel lists every entry, the large-hull
    mode forwards them and the int64 instantiation solves them -- the hand-off path with every
    entry listed); every entry against the oracle's CHT, bit-exact."""
    import dataclasses
    cfg = dataclasses.replace(wl.CONFIGS["W5"], dense_n=(120000, 180000))
    H = wl.make_dense_hist(cfg, seed=0, device=dev)
    ws = torch.empty(sp.place_checkpoints_workspace_bytes(cfg.n_entries, cfg.N, cfg.M),
                     dtype=torch.uint8, device=dev)
    pos, npos, cost, cbb = sp.place_checkpoints(H, cfg.M, cost_by_budget=True, workspace=ws)
    torch.cuda.synchronize()
    st = sp.dp_stats(ws)
    assert st["entries_i64"] == cfg.n_entries and st["entries_hull"] == cfg.n_entries
    pos, npos, cost, cbb = np_(pos), np_(npos), np_(cost), np_(cbb)
    Hc = np_(H)
    del H
    rpos, rnpos, rcost, rcbb = oracle.place_batch(Hc, cfg.M, "cht", nthreads=os.cpu_count() or 1,
                                                  with_budget=True)
    assert (npos == rnpos).all() and (pos == rpos).all()
    assert (cost == rcost).all() and (cbb == rcbb).all()


def test_dp_edge_cases(dev):
    N = 50
    H = np.zeros((8, N + 1), np.int64)
    H[1, 50] = 5                     # point mass at N
    H[2, 1] = 3                      # point mass at 1
    H[3, [3, 10, 40]] = [2, 1, 7]    # K = 3 < M
    H[4, 1:] = 1                     # uniform
    H[5, 0] = 100                    # only misses -> like all-zero
    H[6, 1:] = np.arange(1, N + 1)   # increasing
    H[7, 25] = 1
    for M in (0, 1, 4, 50):
        pos, npos, cost, cbb = gpu_place(H, M, dev)
        check_against_oracle(H, M, pos, npos, cost, cbb, algo="naive")
    # N = 1
    H1 = np.array([[0, 3], [2, 0]], np.int64)
    for M in (0, 1):
        pos, npos, cost, cbb = gpu_place(H1, M, dev)
        check_against_oracle(H1, M, pos, npos, cost, cbb, algo="naive")


def test_dp_wide_path_and_int64_weights(dev):
    """Counts large enough that 2 n N >= 2^31 take the int64 path (still exact)."""
    N, M, E = 3000, 12, 6
    cfg = wl.TraceConfig("t", E, N, M, 1, (N, N), (1, 1), "uniform", dense_n=(N, 2 * N))
    H = wl.make_dense_hist(cfg, seed=9).numpy().astype(np.int64) * 50000
    assert (H.sum(1) * N * 2 >= 2 ** 31).all()
    for dt in (torch.int32, torch.int64):
        pos, npos, cost, cbb = gpu_place(H, M, dev, dtype=dt)
        check_against_oracle(H, M, pos, npos, cost, cbb)
    H64 = H.copy()
    H64[0] *= 2 ** 20                 # int64 weights beyond int32
    pos, npos, cost, cbb = gpu_place(H64, M, dev, dtype=torch.int64)
    check_against_oracle(H64, M, pos, npos, cost, cbb, rows=[0])


def test_dp_wide_path_large_N(dev):
    """int64 path with N beyond the shared-memory limit (b in global/L2 scratch)."""
    N, M, E = 32768, 8, 3
    cfg = wl.TraceConfig("t", E, N, M, 1, (N, N), (1, 1), "mix", dense_n=(60000, 70000))
    H = wl.make_dense_hist(cfg, seed=10).numpy()
    assert (H.sum(1) * N * 2 >= 2 ** 31).all()
    pos, npos, cost, cbb = gpu_place(H, M, dev)
    check_against_oracle(H, M, pos, npos, cost, cbb)


def test_dp_status_flags(dev):
    N, M = 40, 3
    H = np.ones((3, N + 1), np.int64)
    H[1, 7] = -1                               # negative count -> BAD_ARGUMENT for that entry
    H[2, 5] = 2 ** 62 // N                     # 2 n N >= 2^62 -> OVERFLOW for that entry
    pos, npos, cost, cbb = gpu_place(H, M, dev, dtype=torch.int64)
    assert npos[0] == 3
    assert npos[1] == -sp.SP_ERR_BAD_ARGUMENT
    assert npos[2] == -sp.SP_ERR_OVERFLOW
    with pytest.raises(sp.SPError):
        sp.place_checkpoints(torch.ones(2, 5, dtype=torch.int32, device=dev), 5)   # M > N


def test_dp_workspace_too_small(dev):
    w = torch.ones(4, 101, dtype=torch.int32, device=dev)
    with pytest.raises(sp.SPError, match="WORKSPACE"):
        sp.place_checkpoints(w, 4, workspace=torch.empty(16, dtype=torch.uint8, device=dev))


# ------------------------------------------------------------------------------------------
# a7 : fp64 variant
# ------------------------------------------------------------------------------------------


@pytest.mark.parametrize("N,M,E,dyadic", [(500, 7, 10, False), (2048, 8, 8, True),
                                          (8192, 16, 4, False), (4096, 64, 6, False),
                                          (700, 100, 4, False)])
def test_dp_f64_relerr(dev, N, M, E, dyadic):
    """fp64 weights w = c / n (a7): cost and V_0..V_M against the oracle's exact V_int / n at the
    1e-12 bound, the returned positions re-scored by the oracle's fp64 walk; M = 64 (two slots)
    and M = 100 (two chained passes: the e-row buffers then hold the prefix sums)."""
    cfg = wl.TraceConfig("t", E, N, M, 1, (N, N), (1, 1), "mix",
                         dense_n=(4096, 4096) if dyadic else (3000, 9000))
    H = wl.make_dense_hist(cfg, seed=11).numpy().astype(np.int64)
    n = H.sum(1, keepdims=True)
    W = H / n
    pos, npos, cost, cbb = gpu_place(W, M, dev, dtype=torch.float64)
    for e in range(E):
        _, vint, rcbb = oracle.place(H[e], M, "cht")
        ref = vint / n[e, 0]
        assert abs(cost[e] - ref) <= 1e-12 * ref, (e, cost[e], ref)
        # the returned positions achieve it under the oracle's definitional fp64 walk
        got = oracle.expected_cost_f64(W[e], pos[e, :npos[e]])
        assert abs(got - ref) <= 1e-12 * ref
        # V_0..V_M (definitional costs of every budget's canonical placement): the a7 bound
        assert f64_within(cbb[e], rcbb / n[e, 0], H[e]).all(), e


def test_dp_f64_small_vs_f64_oracle(dev):
    rng = np.random.default_rng(12)
    W = rng.random((20, 41)) * (rng.random((20, 41)) < 0.5)
    W[:, 0] = 0
    pos, npos, cost, cbb = gpu_place(W, 5, dev, dtype=torch.float64)
    for e in range(20):
        D, O = oracle.dp_f64(W[e], 5)
        ref = D[5, -1]
        assert abs(cost[e] - ref) <= 1e-12 * max(ref, 1e-300) + 1e-15


# ------------------------------------------------------------------------------------------
# a6 : baseline evaluation
# ------------------------------------------------------------------------------------------


def test_expected_recompute_baselines(dev):
    cfg = wl.scaled(wl.CONFIGS["W4"], 40)
    H = wl.make_dense_hist(cfg, seed=13)
    N = cfg.N
    pos, npos, labels = sp.baseline_sets(N, budgets=range(0, 65), blocks=(64, 128), device=dev)
    cost, worst = sp.expected_recompute(H.to(dev), pos, npos, broadcast=True)
    torch.cuda.synchronize()
    rc, rw = oracle.eval_batch(np_(H), np_(pos), np_(npos), broadcast=True, nthreads=8)
    assert (np_(cost) == rc).all() and (np_(worst) == rw).all()
    # Thm 1.2 / Table 1 tail for balanced: worst = ceil((N+1)/(M+1)) - 1
    for i, (kind, m) in enumerate(labels):
        if kind == "balanced":
            assert (np_(worst)[:, i] == -(-(N + 1) // (m + 1)) - 1).all()


def test_expected_recompute_prefix_widths(dev):
    """int32 rows through both shared-prefix widths (2-byte, 4-byte: SP_DBG_EVAL_PATH) and
    rows whose 1024-bin segments hold >= 2^16 (resp. >= 2^31 in total) counts, which take the
    exact global-memory path, against the oracle's definitional walk."""
    import os
    cfg = wl.scaled(wl.CONFIGS["W5"], 12)
    H = wl.make_dense_hist(cfg, seed=14).numpy()
    H[3, 5000] = 70000                      # one segment >= 2^16
    H[7, 1:2000] = 2 ** 20                  # segments >= 2^31
    N = cfg.N
    pos, npos, _ = sp.baseline_sets(N, budgets=(1, 7, 64), blocks=(64, 128), device=dev)
    rc, rw = oracle.eval_batch(H, np_(pos), np_(npos), broadcast=True, nthreads=8)
    for path in (0, 3, 2, 1):   # automatic (broadcast tables), 2-byte / 4-byte prefixes, chunked
        with sp.debug(SP_DBG_EVAL_PATH=path):
            cost, worst = sp.expected_recompute(torch.from_numpy(H).to(dev), pos, npos,
                                                broadcast=True)
            torch.cuda.synchronize()
        assert (np_(cost) == rc).all() and (np_(worst) == rw).all(), path


@pytest.mark.parametrize("N,E", [(32768, 12), (5, 37), (1000, 301)])
def test_expected_recompute_broadcast_tables(dev, N, E):
    """The broadcast path (<= 4 shared sets: per-CTA l(t; C) tables, one streaming pass per row)
    against the oracle: W5-like and ragged shapes (entry counts not a multiple of the warps per
    CTA, rows not a multiple of the warp width), an empty set, a malformed set, large counts; and
    the same rows through a pointer that is not 16-byte aligned."""
    import dataclasses
    cfg = dataclasses.replace(wl.scaled(wl.CONFIGS["W5"], E), N=N)
    rng = np.random.default_rng(N + E)
    H = rng.integers(0, 50, size=(E, N + 1)).astype(np.int32)
    H[rng.random((E, N + 1)) < 0.7] = 0
    if N >= 1000:
        H[:min(E, 4)] = wl.make_dense_hist(dataclasses.replace(cfg, N=N), seed=3).numpy()[:min(E, 4)]
        H[1, 1:min(N, 2000)] = 2 ** 20           # large counts: int64 sums
    sets = [sp.balanced_positions(N, min(N, 64)), [], sp.block_positions(N, max(1, N // 7))]
    S = len(sets) + 1
    width = max(len(s) for s in sets) + 1
    pos = np.zeros((S, width), np.int32)
    npos = np.zeros(S, np.int32)
    for i, s in enumerate(sets):
        pos[i, :len(s)] = s
        npos[i] = len(s)
    pos[3, :2] = [min(3, N), min(3, N)]        # malformed: not strictly increasing
    npos[3] = 2
    rc, rw = oracle.eval_batch(H, np.ascontiguousarray(pos[:3]), npos[:3], broadcast=True,
                               nthreads=8)   # (the oracle rejects malformed sets outright)
    Hd = torch.from_numpy(H).to(dev)
    for Hin in (Hd, torch.empty(E * (N + 1) + 1, dtype=torch.int32, device=dev)[1:].view(E, N + 1)):
        Hin.copy_(Hd)
        for S in (1, 2, 3, 4):   # every instantiation of the kernel (S is a template parameter)
            cost, worst = sp.expected_recompute(Hin, torch.from_numpy(pos[:S].copy()).to(dev),
                                                torch.from_numpy(npos[:S].copy()).to(dev),
                                                broadcast=True)
            torch.cuda.synchronize()
            k = min(S, 3)
            assert (np_(cost)[:, :k] == rc[:, :k]).all() and (np_(worst)[:, :k] == rw[:, :k]).all()
            if S == 4:
                assert (np_(cost)[:, 3] == -1).all()
                assert (np_(worst)[:, 3] == -sp.SP_ERR_BAD_POSITIONS).all()


@pytest.mark.parametrize("N", [383, 384, 385, 1000])
def test_expected_recompute_bcast_fast_path_thresholds(dev, N):
    """eval_bcast_kernel's uint32 slice sums hold while every count of a 384-bin slice lies in
    [0, 2^13): counts at 2^13 - 1 (fast), 2^13 (int64 path), negative counts and INT32_MAX (int64
    path) are mixed per slice, rows ragged against the slice width; against the oracle."""
    E = 37
    rng = np.random.default_rng(N)
    H = rng.integers(0, 2 ** 13, size=(E, N + 1)).astype(np.int64)
    H[rng.random((E, N + 1)) < 0.5] = 0
    H[:, 0] = rng.integers(0, 5, size=E)                    # bin 0 (misses) is never weighted
    H[1, :] = 2 ** 13 - 1                                   # the fast path's largest count
    H[2, rng.integers(1, N + 1, size=3)] = 2 ** 13          # one count past it per few slices
    H[3, rng.integers(1, N + 1, size=5)] = -1               # negative counts (int64 path)
    H[4, N] = 2 ** 31 - 1                                   # the last bin, INT32_MAX
    H[5, 1:] = 2 ** 31 - 1                                  # a full row of INT32_MAX
    H = H.astype(np.int32)
    sets = [sp.balanced_positions(N, 64), sp.block_positions(N, 64), sp.block_positions(N, 128)]
    width = max(len(x) for x in sets)
    pos = np.zeros((3, width), np.int32)
    npos = np.array([len(x) for x in sets], np.int32)
    for i, x in enumerate(sets):
        pos[i, :len(x)] = x
    rc, rw = oracle.eval_batch(H, pos, npos, broadcast=True, nthreads=8)
    cost, worst = sp.expected_recompute(torch.from_numpy(H).to(dev), torch.from_numpy(pos).to(dev),
                                        torch.from_numpy(npos).to(dev), broadcast=True)
    torch.cuda.synchronize()
    assert (np_(cost) == rc).all() and (np_(worst) == rw).all()


def test_expected_recompute_staged_sweep_sets(dev):
    """eval_p32_kernel with the broadcast sets staged in shared memory (W4's 66-set budget
    sweep, plus an empty and a malformed set): every cost and worst case against the oracle."""
    cfg = wl.scaled(wl.CONFIGS["W4"], 45)
    H = wl.make_dense_hist(cfg, seed=21).numpy()
    pos, npos, _ = sp.baseline_sets(cfg.N, budgets=cfg.M_sweep, blocks=(64, 128), device=dev)
    P = np.zeros((pos.shape[0] + 2, pos.shape[1]), np.int32)
    K = np.zeros(pos.shape[0] + 2, np.int32)
    P[:-2], K[:-2] = np_(pos), np_(npos)
    K[-2] = 0                                   # empty set: cost T_N, worst N
    P[-1, :3] = [10, 9, 30]                     # malformed
    K[-1] = 3
    rc, rw = oracle.eval_batch(H, P[:-1].copy(), K[:-1].copy(), broadcast=True, nthreads=8)
    cost, worst = sp.expected_recompute(torch.from_numpy(H).to(dev), torch.from_numpy(P).to(dev),
                                        torch.from_numpy(K).to(dev), broadcast=True)
    torch.cuda.synchronize()
    assert (np_(cost)[:, :-1] == rc).all() and (np_(worst)[:, :-1] == rw).all()
    assert (np_(cost)[:, -1] == -1).all()
    assert (np_(worst)[:, -1] == -sp.SP_ERR_BAD_POSITIONS).all()


def test_expected_recompute_dp_positions_and_bad_sets(dev):
    """E[r](DP output) == V_M, per-entry (non-broadcast) sets, malformed sets flagged."""
    cfg = wl.scaled(wl.CONFIGS["W3"], 16)
    cfg = wl.TraceConfig(**{**cfg.__dict__, "dense_n": (2000, 5000)})
    H = wl.make_dense_hist(cfg, seed=14).to(dev)
    pos, npos, cost, _ = sp.place_checkpoints(H, 16)
    E, S = 16, 2
    P = torch.zeros(E, S, 16, dtype=torch.int32, device=dev)
    K = torch.zeros(E, S, dtype=torch.int32, device=dev)
    P[:, 0] = pos
    K[:, 0] = npos
    P[:, 1, :3] = torch.tensor([5, 5, 9], dtype=torch.int32)    # not strictly increasing
    K[:, 1] = 3
    c2, w2 = sp.expected_recompute(H, P, K, broadcast=False)
    torch.cuda.synchronize()
    assert (np_(c2)[:, 0] == np_(cost)).all()
    assert (np_(c2)[:, 1] == -1).all() and (np_(w2)[:, 1] == -sp.SP_ERR_BAD_POSITIONS).all()


def test_expected_recompute_f64(dev):
    cfg = wl.scaled(wl.CONFIGS["W4"], 8)
    H = wl.make_dense_hist(cfg, seed=15).numpy().astype(np.int64)
    W = H / H.sum(1, keepdims=True)
    pos, npos, _ = sp.baseline_sets(cfg.N, budgets=(1, 4, 16, 64), blocks=(64,), device=dev)
    cost, worst = sp.expected_recompute(torch.from_numpy(W).to(dev), pos, npos)
    torch.cuda.synchronize()
    rc, _ = oracle.eval_batch(H.astype(np.int32), np_(pos), np_(npos), broadcast=True)
    ref = rc / H.sum(1, keepdims=True)
    assert np.allclose(np_(cost), ref, rtol=1e-13, atol=0)


@pytest.mark.parametrize("N,budgets,blocks", [(8192, (64,), (64, 128)), (2048, (1, 8, 33), (16,)),
                                               (700, (), (1,))])
def test_expected_recompute_f64_broadcast(dev, N, budgets, blocks):
    """fp64 weights with <= 4 broadcast sets (eval_bcast_f64_kernel: the bench's `--weights f64`
    evaluation): against the oracle's exact integer costs / n at 1e-13 relative, and against the
    chunked double-double kernel (SP_DBG_EVAL_PATH = 1); a bin-0 (miss) weight is ignored; a
    malformed set gives NaN and the flagged worst case."""
    cfg = wl.TraceConfig("t", 37, N, 8, 1, (N, N), (1, 1), "mix", dense_n=(N // 3, N))
    H = wl.make_dense_hist(cfg, seed=N).numpy().astype(np.int64)
    H[5, 1:] = 0
    H[5, N] = 3                                    # a point mass at N
    n = np.maximum(H[:, 1:].sum(1, keepdims=True), 1)
    W = H / n
    W[:, 0] = 1e300                                # misses: ignored by the objective
    pos, npos, _ = sp.baseline_sets(N, budgets=budgets, blocks=blocks, device=dev)
    Wd = torch.from_numpy(W).to(dev)
    cost, worst = sp.expected_recompute(Wd, pos, npos)
    with sp.debug(SP_DBG_EVAL_PATH=1):
        cost1, worst1 = sp.expected_recompute(Wd, pos, npos)
    torch.cuda.synchronize()
    Hz = H.copy()
    Hz[:, 0] = 0
    rc, rw = oracle.eval_batch(Hz.astype(np.int32), np_(pos), np_(npos), broadcast=True)
    assert np.allclose(np_(cost), rc / n, rtol=1e-13, atol=0)
    assert np.allclose(np_(cost), np_(cost1), rtol=1e-15, atol=0)
    assert (np_(worst) == rw).all() and (np_(worst1) == rw).all()
    bad = pos.clone()
    if bad.shape[1] >= 2 and int(npos[0]) >= 2:
        bad[0, 1] = bad[0, 0]                      # not strictly increasing
        c2, w2 = sp.expected_recompute(Wd, bad, npos)
        torch.cuda.synchronize()
        assert np.isnan(np_(c2)[:, 0]).all() and (np_(w2)[:, 0] == -sp.SP_ERR_BAD_POSITIONS).all()
        assert np.allclose(np_(c2)[:, 1:], np_(cost)[:, 1:], rtol=0, atol=0)


# ------------------------------------------------------------------------------------------
# e : multi-GPU, emulated on one GPU ("split requests into R shards, sum histograms,
#     assert identical placements")
# ------------------------------------------------------------------------------------------


@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_multirank_emulation_one_gpu(dev, ranks):
    """The N-rank path of bench.py / dist.HistMerger emulated on one GPU: the requests of a
    QuALITY-like trace routed to `ranks` shards exactly as on N ranks (make_trace(world, rank)),
    each shard's depths from sp_overlap_hist(lcp_out, with_hist=False), the all-gather as a
    concatenation of the padded per-rank buffers, every owner's slice scatter-added with
    sp_accumulate_depths; the owners' histograms and placements must equal the single-rank
    ones bit for bit (per-edge independence P:189-190; integer sums commute)."""
    E = 64
    cfg = wl.scaled(wl.CONFIGS["W3"], E)
    N, M = cfg.N, cfg.M
    full = wl.make_trace(cfg, seed=9, device=dev)
    h_ref, _ = sp.overlap_hist(full["entry_tokens"], full["entry_off"], full["req_tokens"],
                               full["req_off"], full["req_entry"], N, n_entries=E)
    shards = [wl.make_trace(cfg, seed=9, device=dev, world=ranks, rank=r) for r in range(ranks)]
    assert sum(s["req_off"].numel() - 1 for s in shards) == full["req_off"].numel() - 1
    Rmax = max(s["req_off"].numel() - 1 for s in shards)
    g_ent, g_lcp = [], []
    for s in shards:
        R = s["req_off"].numel() - 1
        lcp = torch.full((Rmax,), -1, dtype=torch.int32, device=dev)
        ent = torch.full((Rmax,), -1, dtype=torch.int32, device=dev)
        ent[:R] = s["req_entry"]
        sp.overlap_hist(s["entry_tokens"], s["entry_off"], s["req_tokens"], s["req_off"],
                        s["req_entry"], N, lcp_out=lcp, n_entries=E, with_hist=False)
        g_ent.append(ent)
        g_lcp.append(lcp)
    g_ent, g_lcp = torch.cat(g_ent), torch.cat(g_lcp)       # the all-gather
    E_own = E // ranks
    owners = []
    for o in range(ranks):
        h = torch.zeros(E_own, N + 1, dtype=torch.int32, device=dev)
        sp.accumulate_depths(g_ent, g_lcp, o * E_own, (o + 1) * E_own, N, h)
        owners.append(h)
    merged = torch.cat(owners)
    assert torch.equal(merged, h_ref)
    ref = sp.place_checkpoints(h_ref, M, cost_by_budget=True)
    got = [sp.place_checkpoints(h, M, cost_by_budget=True) for h in owners]
    for i in range(4):
        assert torch.equal(torch.cat([g[i] for g in got]), ref[i])
