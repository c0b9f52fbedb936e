"""Pins for the CPU oracle (oracle/) against facts fixed by the paper and by mathematics.

None of these tests compares the oracle with itself: every check is against a value printed
in SPEC/Table 1 (tests/golden/spec_examples.json, each with its citation), a closed form of
the paper (Thm 1, Thm 1.2, Lemma uniform-gap, Lemma stability), an invariant, brute force on
tiny inputs (an independent pure-Python enumeration pins the C brute force), or the
construction of the synthetic trace (LCP = drawn depth by construction).
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2605_05219_b200 import workload as wl

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def counts_of(lst):
    return np.asarray(lst, dtype=np.int64)


def thm1_value(N, M):
    """N * E[r*] under uniform p: (K-rho) q(q-1)/2 + rho q(q+1)/2."""
    K = M + 1
    q, rho = divmod(N + 1, K)
    return (K - rho) * q * (q - 1) // 2 + rho * q * (q + 1) // 2


def f7_positions(N, M):
    """rule-B positions under uniform mass, c_i = i q + max(0, i - (K - rho))."""
    K = M + 1
    q, rho = divmod(N + 1, K)
    return [i * q + max(0, i - (K - rho)) for i in range(1, M + 1)]


def py_cost(c, C):
    """Definitional objective retyped in Python only for the pure-Python brute force below."""
    tot = 0
    for t in range(1, len(c)):
        l = max([0] + [x for x in C if x <= t])
        tot += int(c[t]) * (t - l)
    return tot


def py_brute(c, M):
    """Pure-Python exhaustive search: min cost, colex-min optimum (tiny N only)."""
    N = len(c) - 1
    best = None
    for k in range(0, M + 1):
        for C in itertools.combinations(range(1, N + 1), k):
            v = py_cost(c, C)
            key = (v, tuple(sorted(C, reverse=True)))
            # colex: compare descending tuples lexicographically; proper prefix first
            if best is None or key < best:
                best = key
    return sorted(best[1]), best[0]


# ------------------------------------------------------------------------------------------
# golden examples (SPEC worked examples / Table 1)
# ------------------------------------------------------------------------------------------


@pytest.mark.parametrize("ex", GOLD["reusable_depth"], ids=lambda e: e["cite"][:20])
def test_golden_reusable_depth(ex):
    # r(t;C) = t - l(t;C) is the cost of a point mass at t
    c = np.zeros(ex["N"] + 1, np.int64)
    c[ex["t"]] = 1
    assert oracle.expected_cost(c, ex["C"]) == ex["t"] - ex["l"]


@pytest.mark.parametrize("ex", GOLD["expected_cost"], ids=lambda e: e["cite"][:20])
def test_golden_expected_cost(ex):
    c = counts_of(ex["counts"])
    assert c.sum() == ex["n"]
    assert oracle.expected_cost(c, ex["C"]) == ex["cost_num"]
    assert oracle.worst_case(len(c) - 1, ex["C"]) == ex["worst"]


@pytest.mark.parametrize("ex", GOLD["balanced"], ids=lambda e: e["cite"][:20])
def test_golden_balanced(ex):
    assert oracle.balanced(ex["N"], ex["M"]).tolist() == ex["C"]


@pytest.mark.parametrize("ex", GOLD["uniform_optimal_cost"], ids=lambda e: e["cite"][:20])
def test_golden_uniform_optimal(ex):
    N, M = ex["N"], ex["M"]
    c = np.ones(N + 1, np.int64)
    c[0] = 0
    _, cost, _ = oracle.place(c, M, "naive")
    assert cost == ex["cost_num"] == thm1_value(N, M)


@pytest.mark.parametrize("ex", GOLD["worst_case_optimal"], ids=lambda e: e["cite"][:20])
def test_golden_worst_case(ex):
    assert oracle.worst_case(ex["N"], oracle.balanced(ex["N"], ex["M"])) == ex["worst"]


@pytest.mark.parametrize("ex", GOLD["block"], ids=lambda e: e["cite"][:20])
def test_golden_block(ex):
    assert oracle.block(ex["N"], ex["B"]).tolist() == ex["C"]


@pytest.mark.parametrize("ex", GOLD["dp_optimal"], ids=lambda e: e["cite"][:20])
@pytest.mark.parametrize("algo", ["naive", "cht"])
def test_golden_dp(ex, algo):
    c = counts_of(ex["counts"])
    pos, cost, _ = oracle.place(c, ex["M"], algo)
    assert pos.tolist() == ex["C"]
    assert cost == ex["cost_num"]
    assert oracle.expected_cost(c, pos) == cost


# ------------------------------------------------------------------------------------------
# closed forms
# ------------------------------------------------------------------------------------------


def test_prefix_uniform_closed_form():
    N = 1000
    c = np.ones(N + 1, np.int64)
    c[0] = 0
    P, T = oracle.prefix(c)
    j = np.arange(N + 1)
    assert (P == j).all() and (T == j * (j + 1) // 2).all()


def test_thm1_all_small():
    """Thm 1 for every N <= 120, M <= N: DP value, balanced value, worst case."""
    for N in range(1, 121):
        c = np.ones(N + 1, np.int64)
        c[0] = 0
        D, O = oracle.dp(c, N, "cht")
        for M in range(0, N + 1):
            v = thm1_value(N, M)
            assert D[M, N] == v, (N, M)
            bal = oracle.balanced(N, M)
            assert oracle.expected_cost(c, bal) == v
            assert oracle.worst_case(N, bal) == -(-(N + 1) // (M + 1)) - 1
            pos = oracle.backtrack(O, c, M)
            assert pos.tolist() == f7_positions(N, M), (N, M)


def test_thm1_naive_matches_closed_form():
    for N in (1, 2, 3, 17, 64, 101):
        c = np.ones(N + 1, np.int64)
        c[0] = 0
        D, _ = oracle.dp(c, min(N, 12), "naive")
        for M in range(0, min(N, 12) + 1):
            assert D[M, N] == thm1_value(N, M)


@pytest.mark.parametrize("N,M", [(2048, 8), (8192, 16), (8192, 64), (32768, 64)])
def test_thm1_large(N, M):
    c = np.ones(N + 1, np.int64)
    c[0] = 0
    pos, cost, cbb = oracle.place(c, M, "cht")
    assert cost == thm1_value(N, M)
    assert [int(x) for x in cbb] == [thm1_value(N, m) for m in range(M + 1)]
    assert pos.tolist() == f7_positions(N, M)
    g = np.diff(np.concatenate([[0], pos, [N + 1]]))
    assert g.max() - g.min() <= 1            # "balanced" (Thm 1 iff)


def test_uniform_gap_lemma():
    """Lemma uniform-gap: N E[r] = sum g_i (g_i - 1) / 2 for any C."""
    rng = np.random.default_rng(1)
    for _ in range(300):
        N = int(rng.integers(1, 200))
        k = int(rng.integers(0, min(N, 12) + 1))
        C = np.sort(rng.choice(np.arange(1, N + 1), size=k, replace=False)).astype(np.int32)
        c = np.ones(N + 1, np.int64)
        c[0] = 0
        g = np.diff(np.concatenate([[0], C, [N + 1]]))
        assert oracle.expected_cost(c, C) == int((g * (g - 1) // 2).sum())
        assert oracle.worst_case(N, C) == int(g.max()) - 1


def test_thm1_2_minimax():
    """Thm 1.2: min over |C| = M of max_t r = ceil((N+1)/(M+1)) - 1, by enumeration."""
    for N in range(1, 11):
        for M in range(0, N + 1):
            best = min(oracle.worst_case(N, np.asarray(C, np.int32))
                       for C in itertools.combinations(range(1, N + 1), M))
            assert best == -(-(N + 1) // (M + 1)) - 1


# ------------------------------------------------------------------------------------------
# brute force (exhaustive) and the pure-Python enumeration that pins it
# ------------------------------------------------------------------------------------------


def test_c_brute_force_matches_pure_python():
    for key in range(60):
        N = 1 + key % 9
        c = wl.random_small_hist(7, N, max_count=4, zero_frac=0.35, key=key).numpy()
        for M in range(0, min(N, 3) + 1):
            pos_c, cost_c = oracle.brute_force(c, M)
            pos_p, cost_p = py_brute(c, M)
            assert cost_c == cost_p and pos_c.tolist() == pos_p, (key, M)


def test_dp_equals_brute_force_small():
    """Thm 2 optimality + rule B = colex-min optimum on all N <= 16."""
    n = 0
    for key in range(400):
        N = 1 + key % 16
        c = wl.random_small_hist(11, N, max_count=6, zero_frac=0.4, key=key).numpy()
        for M in range(0, min(N, 4) + 1):
            bpos, bcost = oracle.brute_force(c, M)
            for algo in ("naive", "cht"):
                pos, cost, _ = oracle.place(c, M, algo)
                assert cost == bcost, (key, M, algo)
                assert pos.tolist() == bpos.tolist(), (key, M, algo, pos, bpos)
            n += 1
    assert n > 1000


def test_dp_equals_brute_force_uniform_characterisation():
    """for uniform mass every brute-force optimum has gaps differing by <= 1."""
    for N in range(1, 13):
        c = np.ones(N + 1, np.int64)
        c[0] = 0
        for M in range(0, min(N, 4) + 1):
            opt = thm1_value(N, M)
            for C in itertools.combinations(range(1, N + 1), M):
                g = np.diff(np.concatenate([[0], C, [N + 1]]))
                is_bal = g.max() - g.min() <= 1
                assert (oracle.expected_cost(c, np.asarray(C, np.int32)) == opt) == is_bal


def test_w1_brute_force():
    """W1 (BASELINE.json configs[0]): N=64, M=4 from 100 synthetic requests, brute-forced over
    all 679,121 subsets of size <= 4."""
    cfg = wl.CONFIGS["W1"]
    tr = wl.make_trace(cfg, seed=0)
    hist, lcp = oracle.lcp_hist(tr["entry_tokens"].numpy(), tr["entry_off"].numpy(),
                                tr["req_tokens"].numpy(), tr["req_off"].numpy(),
                                tr["req_entry"].numpy(), cfg.N)
    c = hist[0].astype(np.int64)
    assert c.sum() == 100
    bpos, bcost = oracle.brute_force(c, cfg.M)
    for algo in ("naive", "cht"):
        pos, cost, _ = oracle.place(c, cfg.M, algo)
        assert cost == bcost and pos.tolist() == bpos.tolist()


# ------------------------------------------------------------------------------------------
# invariants
# ------------------------------------------------------------------------------------------


def _hists(seed, n, N):
    out = []
    for key in range(n):
        out.append(wl.random_small_hist(seed, N, max_count=9, zero_frac=0.5, key=key).numpy())
    return out


@pytest.mark.parametrize("N,M", [(40, 6), (97, 12), (300, 20)])
def test_naive_equals_cht_every_cell(N, M):
    """The paper's O(NM) algorithm (P:760-773 with F6 ties) equals the definition on every
    cell, values and leftmost argmins."""
    for c in _hists(3, 25, N):
        D1, O1 = oracle.dp(c, M, "naive")
        D2, O2 = oracle.dp(c, M, "cht")
        assert (D1 == D2).all() and (O1 == O2).all()


def test_naive_equals_cht_generated_shapes():
    cfg = wl.scaled(wl.CONFIGS["W4"], 4)
    cfg = wl.TraceConfig(**{**cfg.__dict__, "N": 512, "dense_n": (300, 600)})
    H = wl.make_dense_hist(cfg, seed=5).numpy()
    for c in H:
        D1, O1 = oracle.dp(c.astype(np.int64), 10, "naive")
        D2, O2 = oracle.dp(c.astype(np.int64), 10, "cht")
        assert (D1 == D2).all() and (O1 == O2).all()


def test_leftmost_argmin_and_monotone_opt():
    """opt[m][j] is the leftmost minimiser (checked against the row recomputed from the w
    definition, independent of the oracle's loop) and non-decreasing in j."""
    for c in _hists(4, 10, 60):
        D, O = oracle.dp(c, 5, "naive")
        N = len(c) - 1
        for m in range(1, 6):
            assert (np.diff(O[m, 1:]) >= 0).all()
            for j in range(1, N + 1):
                vals = [D[m - 1, s - 1] + sum(int(c[t]) * (t - s) for t in range(s, j + 1))
                        for s in range(1, j + 1)]
                assert D[m, j] == min(vals)
                assert O[m, j] == 1 + vals.index(min(vals))


def test_monotone_in_budget_and_dominance():
    """V_m non-increasing in m (BJ) and DP <= balanced / block at equal slots."""
    for c in _hists(5, 30, 150):
        N = len(c) - 1
        M = 16
        _, _, cbb = oracle.place(c, M, "cht")
        assert (np.diff(cbb) <= 0).all()
        assert cbb[0] == oracle.prefix(c)[1][-1]                # V_0 = T_N = n R_nc
        for m in range(0, M + 1):
            assert cbb[m] <= oracle.expected_cost(c, oracle.balanced(N, m))
        for B in (8, 16, 32, 64):
            blk = oracle.block(N, B)
            if len(blk) <= M:
                assert cbb[len(blk)] <= oracle.expected_cost(c, blk)


def test_support_rule():
    """V_M = 0 iff M >= K (K = #mass points); then positions = support."""
    rng = np.random.default_rng(2)
    for _ in range(200):
        N = int(rng.integers(5, 120))
        K = int(rng.integers(1, 8))
        sup = np.sort(rng.choice(np.arange(1, N + 1), size=min(K, N), replace=False))
        c = np.zeros(N + 1, np.int64)
        c[sup] = rng.integers(1, 50, size=sup.size)
        for M in range(0, min(N, 10) + 1):
            pos, cost, _ = oracle.place(c, M, "cht")
            assert (cost == 0) == (M >= sup.size)
            assert len(pos) <= min(M, sup.size)
            assert all(c[p] > 0 for p in pos)                   # every position is a mass point
            if M >= sup.size:
                assert pos.tolist() == sup.tolist()


def test_scale_invariance():
    for c in _hists(6, 20, 80):
        p1, v1, _ = oracle.place(c, 7, "cht")
        p2, v2, _ = oracle.place(c * 13, 7, "cht")
        assert p1.tolist() == p2.tolist() and v2 == 13 * v1


def test_dp_value_equals_definitional_cost():
    """V_M = E[r](returned C) under the definitional walk."""
    for c in _hists(8, 40, 200):
        for M in (1, 3, 9, 25):
            pos, cost, _ = oracle.place(c, M, "cht")
            assert oracle.expected_cost(c, pos) == cost


def test_stability_lemma():
    """Lemma stability: |E_p[r] - E_q[r]| <= N ||p - q||_1."""
    rng = np.random.default_rng(3)
    for _ in range(2000):
        N = int(rng.integers(1, 60))
        p = rng.random(N + 1); p[0] = 0; p /= p.sum()
        q = rng.random(N + 1); q[0] = 0; q /= q.sum()
        k = int(rng.integers(0, N + 1))
        C = np.sort(rng.choice(np.arange(1, N + 1), size=k, replace=False)).astype(np.int32)
        d = abs(oracle.expected_cost_f64(p, C) - oracle.expected_cost_f64(q, C))
        assert d <= N * np.abs(p - q).sum() + 1e-12


# ------------------------------------------------------------------------------------------
# fp64 variant reference
# ------------------------------------------------------------------------------------------


def test_f64_naive_matches_exact_rational():
    """fp64 DP on w = c / n matches V_int / n (exact rational, rounded once) to 1e-15."""
    for c in _hists(9, 15, 120):
        n = c.sum()
        if n == 0:
            continue
        w = c / n
        for M in (0, 2, 7):
            D, O = oracle.dp_f64(w, M)
            _, vint, _ = oracle.place(c, M, "naive")
            ref = vint / n
            assert abs(D[M, -1] - ref) <= 1e-15 * max(ref, 1.0)


# ------------------------------------------------------------------------------------------
# LCP + histogram: the generator fixes the answer by construction
# ------------------------------------------------------------------------------------------


@pytest.mark.parametrize("name,E", [("W1", 1), ("W2", 6), ("W3", 5)])
def test_lcp_hist_equals_construction(name, E):
    cfg = wl.scaled(wl.CONFIGS[name], E)
    tr = wl.make_trace(cfg, seed=1)
    hist, lcp = oracle.lcp_hist(tr["entry_tokens"].numpy(), tr["entry_off"].numpy(),
                                tr["req_tokens"].numpy(), tr["req_off"].numpy(),
                                tr["req_entry"].numpy(), cfg.N, nthreads=2)
    d = np.minimum(tr["depth"].numpy(), cfg.N)
    assert (lcp == d).all()
    ref = np.zeros((E, cfg.N + 1), np.int64)
    np.add.at(ref, (tr["req_entry"].numpy(), d), 1)
    assert (hist == ref).all()


def test_lcp_clamp_and_misses():
    """Depth clamp to N and bin-0 misses, on a hand-built trace."""
    ent = np.array([5, 6, 7, 8, 9, 10], np.int32)
    eoff = np.array([0, 6], np.int64)
    req = np.array([5, 6, 7, 8, 9, 10, 11,   99,   5, 6, 1], np.int32)
    roff = np.array([0, 7, 8, 11], np.int64)
    hist, lcp = oracle.lcp_hist(ent, eoff, req, roff, np.zeros(3, np.int32), N=4)
    assert lcp.tolist() == [4, 0, 2]
    assert hist[0].tolist() == [1, 0, 1, 0, 1]


# ------------------------------------------------------------------------------------------
# structural properties the CUDA D&C relies on (readings R6 / SURVEY F2)
# ------------------------------------------------------------------------------------------


def _structure_cases():
    cases = []
    for key in range(120):
        N = 5 + (key * 37) % 180
        z = [0.0, 0.3, 0.7, 0.95][key % 4]
        cases.append(wl.random_small_hist(41, N, max_count=9, zero_frac=z, key=key).numpy())
    for N in (33, 100, 257):
        c = np.ones(N + 1, np.int64)
        c[0] = 0
        cases.append(c)
    cfg = wl.TraceConfig("s", 6, 700, 12, 1, (700, 700), (1, 1), "uniform", dense_n=(300, 2000))
    cases += list(wl.make_dense_hist(cfg, seed=8).numpy().astype(np.int64))
    return cases


def test_leftmost_argmin_monotone_across_layers():
    """opt_{m-1}(j) <= opt_m(j) for the leftmost argmins (used by the kernel as a lower bracket
    bound; the kernel also flags any empty bracket as SP_ERR_INTERNAL)."""
    for c in _structure_cases():
        N = len(c) - 1
        M = min(N, 16)
        _, O = oracle.dp(c, M, "cht")
        for m in range(2, M + 1):
            assert (O[m, 1:] >= O[m - 1, 1:]).all(), (N, m)


def test_dp_monge_in_budget_and_prefix():
    """dp[k][a] + dp[k+1][b] <= dp[k][b] + dp[k+1][a] for a < b (the marginal value of one more
    checkpoint grows with the prefix), the property behind the layer monotonicity above."""
    for c in _structure_cases()[::3]:
        N = len(c) - 1
        M = min(N, 10)
        D, _ = oracle.dp(c, M, "cht")
        for k in range(0, M):
            d = D[k] - D[k + 1]            # non-decreasing in the prefix length
            assert (np.diff(d) >= 0).all(), (N, k)


def test_row_argmin_monotone_in_j_sparse():
    """SURVEY F2 on sparse/zero-heavy histograms too: opt_m(j) non-decreasing in j."""
    for c in _structure_cases():
        N = len(c) - 1
        _, O = oracle.dp(c, min(N, 12), "cht")
        assert (np.diff(O[1:, 1:], axis=1) >= 0).all()


def test_expected_cost_f64_pins():
    """or_expected_cost_f64 (P:171-173 on fp64 weights) pinned independently of itself:
    (1) a point mass at depth d costs exactly d - l(d; C), l = the largest position <= d (0 if
    none) -- the textbook reusable depth of P:133-137, restated here in plain Python, so an
    off-by-one in r(t) or in l fails; (2) weights c / 2^k with a dyadic total are exact in
    binary, so the fp64 cost equals the integer oracle's cost / 2^k bit for bit."""
    rng = np.random.default_rng(5)
    N = 40
    for _ in range(30):
        k = int(rng.integers(0, 6))
        C = np.sort(rng.choice(np.arange(1, N + 1), size=k, replace=False)).astype(np.int32)
        for d in range(1, N + 1):
            w = np.zeros(N + 1)
            w[d] = 1.0
            l = max([c for c in C.tolist() if c <= d], default=0)
            assert oracle.expected_cost_f64(w, C) == d - l
    for _ in range(30):
        c = rng.integers(0, 50, N + 1).astype(np.int64)
        c[0] = 0
        total = 1 << int(np.ceil(np.log2(max(2, c.sum() + 1))))
        c[N] += total - c.sum()
        assert c.sum() == total
        k = int(rng.integers(0, 8))
        C = np.sort(rng.choice(np.arange(1, N + 1), size=k, replace=False)).astype(np.int32)
        assert oracle.expected_cost_f64(c / total, C) == oracle.expected_cost(c, C) / total
