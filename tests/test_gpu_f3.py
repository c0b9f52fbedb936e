"""f3 parity: the all-budget frontier (the budget sweeps of Figs. 2-3,
P:420-454).  One DP at M_max must return, for every m <= M_max, exactly the canonical (rule B)
placement and cost an m-layer run returns -- checked against the oracle's own m-layer DP."""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_05219_b200 import sp
from paper_2605_05219_b200 import workload as wl

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    sp.lib()
    return torch.device("cuda:0")


def frontier(H, M, dev, dtype=torch.int32):
    w = torch.as_tensor(H).to(dtype).to(dev).contiguous()
    fpos, fn, cbb = sp.place_checkpoints_frontier(w, M)
    torch.cuda.synchronize()
    return fpos.cpu().numpy(), fn.cpu().numpy(), cbb.cpu().numpy()


def check(H, M, fpos, fn, cbb, rows=None, algo="cht"):
    for e in (range(H.shape[0]) if rows is None else rows):
        c = H[e].astype(np.int64)
        D, O = oracle.dp(c, M, algo)
        assert (cbb[e] == D[:, -1]).all(), e
        for m in range(1, M + 1):
            # the oracle's OWN m-layer run (not a slice of its M-layer table)
            rp, rc, _ = oracle.place(c, m, algo)
            k = len(rp)
            assert fn[e, m - 1] == k, (e, m, fn[e, m - 1], k)
            assert fpos[e, m - 1, :k].tolist() == rp.tolist(), (e, m)
            assert (fpos[e, m - 1, k:] == 0).all()
            assert oracle.expected_cost(c, rp) == rc == cbb[e, m]


def test_frontier_small_exhaustive(dev):
    for N in (1, 2, 5, 9, 16):
        H = np.stack([wl.random_small_hist(21, N, max_count=6, zero_frac=z, key=k).numpy()
                      for k, z in enumerate([0.0, 0.3, 0.6, 0.9] * 3)])
        fpos, fn, cbb = frontier(H, N, dev)
        check(H, N, fpos, fn, cbb, algo="naive")


@pytest.mark.parametrize("N,M,E", [(300, 20, 6), (2048, 32, 4)])
def test_frontier_dense(dev, N, M, E):
    cfg = wl.TraceConfig("t", E, N, M, 1, (N, N), (1, 1), "uniform", dense_n=(N // 2, 4 * N))
    H = wl.make_dense_hist(cfg, seed=N + 3).numpy()
    fpos, fn, cbb = frontier(H, M, dev)
    check(H, M, fpos, fn, cbb)


def test_frontier_w4_shape_sampled(dev):
    """W4's budget sweep (M up to 64) on W4-shaped histograms, int64 weights (wide path)."""
    cfg = wl.scaled(wl.CONFIGS["W4"], 8)
    H = wl.make_dense_hist(cfg, seed=21).numpy()
    fpos, fn, cbb = frontier(H, 64, dev, dtype=torch.int64)
    check(H, 64, fpos, fn, cbb, rows=[0, 5])


def test_frontier_sparse_support_and_zero(dev):
    """Support smaller than the budget: budgets past |supp| stop early (rule B); all-zero rows
    give empty sets for every budget."""
    N, M = 50, 8
    H = np.zeros((3, N + 1), np.int32)
    H[0, [7, 30]] = [5, 2]
    H[1, 50] = 1
    fpos, fn, cbb = frontier(H, M, dev)
    check(H, M, fpos, fn, cbb, algo="naive")
    assert (fn[2] == 0).all() and (cbb[2] == 0).all()
    assert fn[0].tolist() == [1] + [2] * 7


def test_frontier_f64_consistent_with_single_runs(dev):
    """fp64 variant: each budget's frontier row achieves the oracle's fp64 optimum for that m."""
    rng = np.random.default_rng(5)
    W = rng.random((6, 201)) * (rng.random((6, 201)) < 0.4)
    W[:, 0] = 0
    M = 10
    fpos, fn, cbb = frontier(W, M, dev, dtype=torch.float64)
    for e in range(W.shape[0]):
        D, _ = oracle.dp_f64(W[e], M)
        for m in range(1, M + 1):
            got = oracle.expected_cost_f64(W[e], fpos[e, m - 1, :fn[e, m - 1]])
            assert abs(got - D[m, -1]) <= 1e-12 * max(D[m, -1], 1e-300) + 1e-15, (e, m)
