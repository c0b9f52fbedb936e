"""Oracle pins for f2: Thm 4's exponentially weighted empirical histogram and its
variance term, against values the paper/SPEC fix and against independent computations (the
online recursion w <- g w + e_T, the geometric-series normaliser, the empirical distribution at
g = 1, the exact sum of squared weights)."""
import numpy as np
import pytest

import oracle


def test_spec_example_gamma_half():
    # g = 0.5, observations (2, 2, 5), N = 5 -> p = [0, 0, 3/7, 0, 0, 4/7]
    # (weights g^(t-s) = 1/4, 1/2, 1 normalised by (1-g)/(1-g^3) = 4/7)
    p = oracle.gamma_hist([2, 2, 5], 5, 0.5)
    assert np.allclose(p, [0, 0, 3 / 7, 0, 0, 4 / 7], rtol=0, atol=1e-15)


def test_point_mass_and_empirical():
    assert np.array_equal(oracle.gamma_hist([3], 6, 0.9), np.eye(7)[3])
    d = np.array([1, 1, 2, 2, 4, 6, 6, 6])
    p = oracle.gamma_hist(d, 6, 1.0)                                         # S:290, Thm 3
    assert np.allclose(p, np.bincount(d, minlength=7) / d.size, rtol=0, atol=1e-15)
    rng = np.random.default_rng(0)
    assert np.allclose(oracle.gamma_hist(rng.permutation(d), 6, 1.0), p, atol=1e-15)


@pytest.mark.parametrize("g", [0.3, 0.9, 0.99])
def test_matches_online_recursion(g):
    """The definition equals the online update w <- g w + e_T normalised by its total,
    and the total equals the geometric series (1 - g^t) / (1 - g)."""
    rng = np.random.default_rng(1)
    N, t = 40, 300
    d = rng.integers(0, N + 3, t)      # includes depths beyond N (clamped) and misses (0)
    w = np.zeros(N + 1)
    h = 0
    for x in d:
        if x < 1:                      # a miss is not a sample of T in {1..N} (R15)
            continue
        w *= g
        w[min(x, N)] += 1.0
        h += 1
    assert abs(w.sum() - (1 - g ** h) / (1 - g)) < 1e-9 * w.sum()
    p = oracle.gamma_hist(d, N, g)
    assert np.allclose(p, w / w.sum(), rtol=1e-12, atol=1e-15)
    assert abs(p.sum() - 1) < 1e-12


def test_order_sensitivity():
    a = oracle.gamma_hist([1, 2], 3, 0.8)
    b = oracle.gamma_hist([2, 1], 3, 0.8)
    assert not np.allclose(a, b) and np.allclose(a[[1, 2]], b[[2, 1]])


def test_variance_term():
    N = 100
    assert abs(oracle.gamma_variance_term(0.99, 1, N) - np.sqrt(N)) < 1e-12
    assert abs(oracle.gamma_variance_term(0.99, 10 ** 6, N) - 0.709) < 1e-3
    for g, t in [(0.5, 7), (0.9, 50), (0.99, 400)]:
        s = np.arange(1, t + 1)
        wts = (1 - g) * g ** (t - s) / (1 - g ** t)
        assert abs(oracle.gamma_variance_term(g, t, N) - np.sqrt(N * (wts ** 2).sum())) < 1e-10
    v = [oracle.gamma_variance_term(0.9, t, N) for t in range(1, 60)]
    assert all(x > y for x, y in zip(v, v[1:]))


def test_thm4_tracking_bound_monte_carlo():
    """Thm 4: E||p_hat - p_t||_1 <= exact bias sum + variance term, for a drifting
    law with known p_s (200 trials)."""
    rng = np.random.default_rng(7)
    N, t, g = 12, 120, 0.9
    base = rng.random(N + 1)
    base[0] = 0
    laws = []
    for s in range(t):
        q = base * (1 + 0.4 * np.sin(0.05 * s + np.arange(N + 1)))
        laws.append(q / q.sum())
    laws = np.array(laws)
    errs = []
    for _ in range(200):
        d = np.array([rng.choice(N + 1, p=laws[s]) for s in range(t)])
        errs.append(np.abs(oracle.gamma_hist(d, N, g) - laws[-1]).sum())
    s = np.arange(1, t + 1)
    wts = (1 - g) * g ** (t - s) / (1 - g ** t)
    bias = (wts * np.abs(laws - laws[-1]).sum(1)).sum()
    assert np.mean(errs) <= bias + oracle.gamma_variance_term(g, t, N)


def test_misses_are_not_samples():
    """Thm 4 samples T_s in {1..N} conditioned on hits (reading R15):
    interleaving misses (depth <= 0) anywhere in the stream leaves the estimate unchanged, bin 0
    stays empty, and a stream of misses only gives the zero vector."""
    rng = np.random.default_rng(7)
    N = 30
    hits = rng.integers(1, N + 4, 200)
    for g in (0.5, 0.9, 1.0):
        ref = oracle.gamma_hist(hits, N, g)
        mixed = hits.tolist()
        for _ in range(80):
            mixed.insert(int(rng.integers(0, len(mixed) + 1)), int(rng.integers(-3, 1)))
        p = oracle.gamma_hist(np.array(mixed), N, g)
        assert np.array_equal(p, ref) and p[0] == 0 and abs(p.sum() - 1) < 1e-12
        # the same via the SPEC example: misses around (2, 2, 5) at g = 0.5
    p = oracle.gamma_hist([0, 2, -1, 2, 0, 5, 0], 5, 0.5)
    assert np.allclose(p, [0, 0, 3 / 7, 0, 0, 4 / 7], rtol=0, atol=1e-15)
    assert np.array_equal(oracle.gamma_hist([0, -2, 0], 5, 0.9), np.zeros(6))
