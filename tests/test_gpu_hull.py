"""GPU parity of the hull kernel (dp_hull.cu: the paper's monotone convex-hull trick, P:764-773,
with all layers in lockstep, one warp per entry) and of its hand-off to the divide-and-conquer
kernel (ring overflow, int64 range, bad counts) -- against the CPU oracle's naive DP (the
definition, Thm 2) or its CHT, bit-exact in every integer output."""
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


def place(H, M, dev, dtype=torch.int32, frontier=False):
    w = torch.as_tensor(H).to(dtype).to(dev).contiguous()
    E, N = w.shape[0], w.shape[1] - 1
    ws = torch.empty(sp.place_checkpoints_workspace_bytes(E, N, M), dtype=torch.uint8, device=dev)
    if frontier:
        fp, fn, cbb = sp.place_checkpoints_frontier(w, M, workspace=ws)
        torch.cuda.synchronize()
        return dict(fpos=np_(fp), fn=np_(fn), cbb=np_(cbb), stats=sp.dp_stats(ws))
    pos, npos, cost, cbb = sp.place_checkpoints(w, M, cost_by_budget=True, workspace=ws)
    torch.cuda.synchronize()
    return dict(pos=np_(pos), npos=np_(npos), cost=np_(cost), cbb=np_(cbb), stats=sp.dp_stats(ws))


def check(H, M, r, algo="cht", rows=None):
    rows = range(H.shape[0]) if rows is None else rows
    for e in rows:
        rp, rc, rcbb = oracle.place(H[e].astype(np.int64), M, algo)
        k = len(rp)
        assert r["npos"][e] == k, (e, r["npos"][e], k)
        assert r["pos"][e, :k].tolist() == rp.tolist(), (e, r["pos"][e, :k], rp)
        assert (r["pos"][e, k:] == 0).all()
        assert r["cost"][e] == rc, (e, r["cost"][e], rc)
        assert (r["cbb"][e] == rcbb).all(), e


def dense(E, N, seed, law="mix", lo=None, hi=None):
    cfg = wl.TraceConfig("t", E, N, 8, 1, (N, N), (1, 1), law,
                         dense_n=(lo or N // 3, hi or N // 2))
    return wl.make_dense_hist(cfg, seed=seed).numpy()


@pytest.mark.parametrize("M", [1, 2, 31, 32, 33, 47, 63, 64])
def test_hull_layer_slots(dev, M):
    """K = 1 (M <= 32) and K = 2 (M > 32, partially filled second slot) against the naive DP."""
    H = dense(12, 600, seed=M)
    r = place(H, M, dev)
    assert r["stats"]["entries_hull"] == 12
    check(H, M, r, algo="naive")


@pytest.mark.parametrize("N,M", [(700, 65), (700, 100), (500, 129), (400, 200), (300, 300)])
def test_hull_multi_pass(dev, N, M):
    """M > 64: passes of 64 layers chained through the e-row buffer."""
    H = dense(6, N, seed=N + M, lo=N // 2, hi=N)
    r = place(H, M, dev)
    assert r["stats"]["entries_hull"] + r["stats"]["entries_i64"] >= 1
    check(H, M, r, algo="cht")


def test_hull_sparse_ties_and_plateaus(dev):
    """Many zero bins (long P_j plateaus: ties between lines), tiny counts, all equal counts."""
    rng = np.random.default_rng(3)
    N, E = 777, 24
    H = np.zeros((E, N + 1), np.int64)
    for e in range(E):
        k = rng.integers(1, 60)
        H[e, rng.integers(1, N + 1, k)] = rng.integers(1, 3, k)
    H[0, :] = 0
    H[1, 1:] = 0
    H[1, N] = 4
    r = place(H, 16, dev)
    check(H, 16, r, algo="naive")
    r = place(H, 64, dev)
    check(H, 64, r, algo="naive")


def test_hull_overflow_falls_back_exactly(dev):
    """Uniform mass: the layer-1 hull holds ~N/2 lines and opt changes every other row, so the
    hull outgrows the shared rings (and the int32 retry's 256-line arrays) and, at N = 3000, a
    change log of max(1024, N/8) entries would fill too: the int32 large-hull mode (unary logs,
    big global arrays) solves both.  Mixed in one batch with dense entries, an int64-range entry
    (int64 hull instantiation) and a bad entry (D&C)."""
    M = 40
    for N in (1000, 3000):
        H = dense(8, N, seed=1).astype(np.int64)
        H[2, 1:] = 1
        H[5, 1:] = 3
        H[6] *= (2 ** 31 // N) // max(1, H[6].sum()) + 1   # n N + T_N >= 2^31: int64 instantiation
        assert H[6].sum() * N >= 2 ** 31 // 2
        r = place(H, M, dev, dtype=torch.int64)
        assert r["stats"]["entries_hull"] == 8
        assert r["stats"]["entries_hull_big"] == 2
        assert r["stats"]["entries_i64"] == 1
        assert r["stats"]["evaluations"] == 0
        check(H, M, r)
        Hb = H.copy()
        Hb[3, 9] = -1
        r = place(Hb, M, dev, dtype=torch.int64)
        assert r["npos"][3] == -sp.SP_ERR_BAD_ARGUMENT
        check(Hb, M, r, rows=[0, 1, 2, 4, 5, 6, 7])


@pytest.mark.parametrize("E", [64, 4000])
def test_hull_int64_list_handoff_all_entries(dev, E):
    """Every entry handed off by the int32 kernel (its list holds all E): half all-ones rows (the
    large-hull mode solves them), half heavy rows past n N + T_N < 2^31 (forwarded by the
    large-hull mode to the int64 instantiation, and from there to the D&C kernel).  The forwarded list has its own array (round 2
    first wrote it into the back of the int64 list's, which overlapped here)."""
    N, M = 4096, 40
    rng = np.random.default_rng(E)
    H = np.zeros((E, N + 1), np.int64)
    H[0::2, 1:] = 1
    H[1::2, 1:] = rng.integers(100, 157, (E // 2, N))           # n ~ 5.2e5: n N ~ 2.1e9
    t = np.arange(N + 1)
    assert (H[1::2, 1:].sum(1) * N + (H[1::2] * t).sum(1) >= 2 ** 31).all()   # past the guard
    r = place(H, M, dev, dtype=torch.int64)
    # the heavy rows are near-uniform: the int64 instantiation's change logs fill, so the D&C
    # kernel solves those it cannot (every output is checked against the oracle below)
    st = r["stats"]
    assert st["entries_hull_big"] == E // 2 and st["entries_i32"] == E // 2
    assert st["entries_i64"] == E // 2   # the int64 hull instantiation or the D&C in int64
    rows = range(E) if E <= 64 else list(range(0, E, 97)) + list(range(1, E, 101))
    check(H, M, r, rows=rows)
    # every heavy row in the batch is the same law: spot-check the rest against its V_M
    if E > 64:
        rp, rc, _ = oracle.place(H[1].astype(np.int64), M, "cht")
        assert r["cost"][1] == rc


@pytest.mark.parametrize("N,M,E", [(2048, 16, 6), (4096, 33, 6), (4096, 64, 40), (32768, 64, 5)])
def test_hull_large_hull_mode(dev, N, M, E):
    """Full-support rows -- all-ones (Thm 1's uniform law; n N + T_N < 2^31 keeps N = 32768 on
    the int32 path) and near-uniform noise in {1, 2, 3} -- have hulls of ~N/(m+1) lines and an
    argmin that moves on most rows: the int32 large-hull mode solves them (no D&C), next to
    sparse W5-like rows on the ordinary kernel; positions, counts, V_M and V_0..V_M against the
    oracle's CHT.  E = 40 runs the one-warp kernel's hand-off, E <= 6 SPLIT's (M > 32)."""
    rng = np.random.default_rng(N + M)
    H = dense(E, N, seed=N + M, lo=N // 8, hi=N // 4).astype(np.int64)
    big = list(range(0, E, 2))
    for e in big:
        H[e, 1:] = 1 if e % 4 == 0 else rng.integers(1, 4, N)
    for dtype in (torch.int32, torch.int64):
        r = place(H, M, dev, dtype=dtype)
        assert r["stats"]["entries_hull"] == E
        # (a noise row's hull may still fit the int32 retry's arrays at small N)
        assert 1 <= r["stats"]["entries_hull_big"] <= len(big)
        assert r["stats"]["evaluations"] == 0
        check(H, M, r)
    # Thm 1: under the uniform law the balanced spacing is optimal -- its cost
    # equals V_M of the all-ones row
    bpos, bnpos, _ = sp.baseline_sets(N, budgets=(M,), blocks=(), device=dev)
    bc, _ = sp.expected_recompute(torch.ones(1, N + 1, dtype=torch.int32, device=dev), bpos, bnpos)
    assert int(bc[0, 0]) == int(r["cost"][0])


def test_hull_matches_dc_kernel_w5_rows(dev):
    """Hull kernel vs the D&C kernel (SP_NO_HULL) on W5-shaped rows at full N=32768, M=64:
    identical positions, counts and every V_m."""
    cfg = wl.scaled(wl.CONFIGS["W5"], 40)
    H = wl.make_dense_hist(cfg, seed=4).numpy()
    a = place(H, 64, dev)
    assert a["stats"]["entries_hull"] == 40
    with sp.debug(SP_DBG_NO_HULL=1):
        b = place(H, 64, dev)
    assert b["stats"]["entries_hull"] == 0
    for k in ("pos", "npos", "cost", "cbb"):
        assert (a[k] == b[k]).all(), k
    check(H, 64, a, rows=[0, 13, 39])


def test_hull_frontier(dev):
    """f3 frontier positions from the hull kernel's argmin table == single-budget oracle runs."""
    H = dense(5, 900, seed=8)
    M = 40
    r = place(H, M, dev, frontier=True)
    assert r["stats"]["entries_hull"] == 5
    for e in range(5):
        for m in (1, 7, 32, 33, 40):
            rp, rc, _ = oracle.place(H[e].astype(np.int64), m, "cht")
            k = len(rp)
            assert r["fn"][e, m - 1] == k
            assert r["fpos"][e, m - 1, :k].tolist() == rp.tolist()
            assert (r["fpos"][e, m - 1, k:] == 0).all()


def test_hull_vs_dc_every_w5_entry(dev):
    """All 16384 W5 entries (the bench launch): hull kernel (incl. its global-ring retries) vs the
    divide-and-conquer kernel alone (SP_NO_HULL) -- identical positions, counts and V_0..V_M."""
    cfg = wl.CONFIGS["W5"]
    H = wl.make_dense_hist(cfg, seed=0, device=dev)
    a = sp.place_checkpoints(H, cfg.M, cost_by_budget=True)
    with sp.debug(SP_DBG_NO_HULL=1):
        b = sp.place_checkpoints(H, cfg.M, cost_by_budget=True)
    torch.cuda.synchronize()
    for x, y, name in zip(a, b, ("pos", "npos", "cost", "cbb")):
        assert torch.equal(x, y), name


def test_hull_int64_path_large_counts(dev):
    """Accumulated histograms beyond the int32 guard (n N >= 2^30, here n ~ 1.5e5 at N = 32768)
    run on the int64 hull instantiation: identical to the D&C kernel on every output, and to
    the oracle's CHT on sampled rows; counts past n N >= 2^46 go to the D&C."""
    import dataclasses
    cfg = dataclasses.replace(wl.scaled(wl.CONFIGS["W5"], 96), dense_n=(120000, 180000))
    H = wl.make_dense_hist(cfg, seed=5).numpy().astype(np.int64)
    H[7] *= 2 ** 14                               # n N >= 2^46: D&C int64
    a = place(H, 64, dev, dtype=torch.int64)
    # hulls of large-n rows outgrow the shared rings more often; the global-ring pool is
    # bounded, so a few entries may reach the D&C -- the outputs are identical either way
    assert a["stats"]["entries_i64"] == 96 and a["stats"]["entries_hull"] >= 80
    with sp.debug(SP_DBG_NO_HULL=1):
        b = place(H, 64, dev, dtype=torch.int64)
    for k in ("pos", "npos", "cost", "cbb"):
        assert (a[k] == b[k]).all(), k
    check(H, 64, a, rows=[0, 7, 50])


def test_hull_f64_path_vs_exact(dev):
    """fp64 weights (a7) on the double hull instantiation at M = 64 (dp_hull_kernel<double, 2,
    double>): W5-shaped rows scaled to probabilities (w = c / n, non-dyadic n).  The exact
    optimum V_int / n comes from the ORACLE's integer CHT; the returned cost and
    every V_0..V_M meet SURVEY 8(c) a7's 1e-12 bound, the returned positions achieve it under the
    oracle's definitional fp64 walk, and the D&C kernel agrees (reading R10)."""
    cfg = wl.scaled(wl.CONFIGS["W5"], 24)
    H = wl.make_dense_hist(cfg, seed=11).numpy().astype(np.int64)
    W = H / H.sum(1, keepdims=True)
    r = place(W, 64, dev, dtype=torch.float64)
    assert r["stats"]["entries_f64"] == 24 and r["stats"]["entries_hull"] >= 20
    _, _, vint, vcbb = oracle.place_batch(H.astype(np.int32), 64, "cht", nthreads=os.cpu_count() or 1,
                                          with_budget=True)
    n = H.sum(1).astype(np.float64)
    for e in range(24):
        assert f64_within([r["cost"][e]], [vint[e] / n[e]], H[e]).all(), e
        assert f64_within(r["cbb"][e], vcbb[e] / n[e], H[e]).all(), e
        got = oracle.expected_cost_f64(W[e], r["pos"][e, :r["npos"][e]])
        assert f64_within([got], [vint[e] / n[e]], H[e]).all(), e
    with sp.debug(SP_DBG_NO_HULL=1):
        d = place(W, 64, dev, dtype=torch.float64)
    for e in range(24):
        assert f64_within([d["cost"][e]], [vint[e] / n[e]], H[e]).all(), e
        assert f64_within(d["cbb"][e], vcbb[e] / n[e], H[e]).all(), e


LOGFULL_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import oracle
from paper_2605_05219_b200 import sp, workload as wl
dev = torch.device('cuda:0')
c = wl.TraceConfig('t', 10, 700, 8, 1, (700, 700), (1, 1), 'mix', dense_n=(233, 350))
H = wl.make_dense_hist(c, seed=21).numpy()
w = torch.as_tensor(H).to(dev).contiguous()
ws = torch.empty(sp.place_checkpoints_workspace_bytes(10, 700, 40), dtype=torch.uint8, device=dev)
pos, npos, cost, cbb = sp.place_checkpoints(w, 40, cost_by_budget=True, workspace=ws)
torch.cuda.synchronize()
assert sp.dp_stats(ws)['entries_hull'] < 10
pos, npos, cost, cbb = (t.cpu().numpy() for t in (pos, npos, cost, cbb))
for e in range(10):
    rp, rc, rcbb = oracle.place(H[e].astype(np.int64), 40, 'naive')
    k = len(rp)
    assert npos[e] == k and pos[e, :k].tolist() == rp.tolist() and cost[e] == rc, e
    assert (cbb[e] == rcbb).all(), e
print('logfull ok')
"""


def run_with_env(script, **env):
    """The library reads its test hooks (SP_HULL_LOGCAP, SP_HULL_LEAN, ...) once per process:
    run the check in a fresh interpreter with them set."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", script, root], env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout + r.stderr


def test_hull_log_full_falls_back(dev):
    """Entries whose argmin-change log fills (forced with a tiny capacity) are solved by the
    D&C kernel instead -- same outputs as the oracle."""
    rc, out = run_with_env(LOGFULL_SCRIPT, SP_HULL_LOGCAP="3")
    assert rc == 0 and "logfull ok" in out, out


LEAN_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import oracle
from paper_2605_05219_b200 import sp, workload as wl
dev = torch.device('cuda:0')
cases = []
cfg = wl.scaled(wl.CONFIGS['W5'], 24)
cases.append((wl.make_dense_hist(cfg, seed=7).numpy(), 64))
for N, M, seed in ((3000, 40, 3), (700, 17, 5), (2048, 8, 6)):
    c = wl.TraceConfig('t', 16, N, M, 1, (N, N), (1, 1), 'mix', dense_n=(N // 4, N // 2))
    cases.append((wl.make_dense_hist(c, seed=seed).numpy(), M))
H = np.zeros((4, 2001), np.int64); H[0, 1:] = 1; H[1, 5] = 9; H[3, ::7] = 2
cases.append((H, 40))   # all-ones (ring overflow -> int64 instantiation), point mass, empty, sparse
for H, M in cases:
    w = torch.as_tensor(H).to(torch.int32).to(dev).contiguous()
    E, N = w.shape[0], w.shape[1] - 1
    ws = torch.empty(sp.place_checkpoints_workspace_bytes(E, N, M), dtype=torch.uint8, device=dev)
    pos, npos, cost, cbb = sp.place_checkpoints(w, M, cost_by_budget=True, workspace=ws)
    torch.cuda.synchronize()
    pos, npos, cost, cbb = (t.cpu().numpy() for t in (pos, npos, cost, cbb))
    for e in range(E):
        rp, rc, rcbb = oracle.place(H[e].astype(np.int64), M, 'cht')
        k = len(rp)
        assert npos[e] == k and pos[e, :k].tolist() == rp.tolist() and cost[e] == rc, (N, M, e)
        assert (cbb[e] == rcbb).all(), (N, M, e)
print('lean ok')
"""


def test_lean_kernel_matches_oracle(dev):
    """dp_lean_kernel (SP_HULL_LEAN=1, read once per process: a subprocess) against the oracle's
    CHT on W5 rows, smaller dense configs, the all-ones row (its ring overflow goes to the int64
    instantiation), a point mass, an empty row and a sparse row."""
    rc, out = run_with_env(LEAN_SCRIPT, SP_HULL_LEAN="1")
    assert rc == 0 and "lean ok" in out, out


ONEWARP_SCRIPT = LEAN_SCRIPT.replace("print('lean ok')", "print('onewarp ok')")


def test_one_warp_mode_on_small_batches(dev):
    """Small batches run in SPLIT mode (two warps per entry) by default; SP_HULL_SPLIT=0 forces
    the one-warp kernel on the same cases -- both against the oracle's CHT."""
    rc, out = run_with_env(ONEWARP_SCRIPT, SP_HULL_SPLIT="0")
    assert rc == 0 and "onewarp ok" in out, out
    rc, out = run_with_env(ONEWARP_SCRIPT.replace("onewarp ok", "split ok"), SP_HULL_SPLIT="1")
    assert rc == 0 and "split ok" in out, out



def test_huge_counts_flag_overflow(dev):
    """int64 counts whose row sum would wrap int64 (four counts of 2^62) or that exceed 2^47
    must come back as -SP_ERR_OVERFLOW (header contract), never as a silent int32-path answer;
    a negative count as -SP_ERR_BAD_ARGUMENT.  The other entries of the batch stay exact."""
    N, M = 40, 5
    H = dense(6, N, seed=31).astype(np.int64)
    H[1, 1:5] = 1 << 62            # sums to 2^64: wraps to 0 in int64
    H[2, 7] = 1 << 48
    H[4, 3] = -1
    r = place(H, M, dev, dtype=torch.int64)
    assert r["npos"][1] == -sp.SP_ERR_OVERFLOW and r["npos"][2] == -sp.SP_ERR_OVERFLOW
    assert r["npos"][4] == -sp.SP_ERR_BAD_ARGUMENT
    check(H, M, r, rows=[0, 3, 5])
