"""GPU parity for f1 (block-aware placement): the block-restricted DP against the oracle's
naive grid DP (positions + int64 costs + V_0..V_M bit-exact), post-hoc clipping against the
oracle's literal clip, and the fp64 grid DP within 1e-12."""
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
        pytest.fail("GPU tests need a CUDA device")
    from paper_2605_05219_b200 import build
    build.build()
    return torch.device("cuda:0")


def np_(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("N,M,B,E", [(50, 3, 4, 20), (300, 8, 7, 12), (1000, 5, 64, 10),
                                     (2048, 8, 64, 8), (4097, 16, 128, 6), (100, 4, 128, 5),
                                     (512, 600 // 100, 1, 4)])
def test_grid_dp_parity(dev, N, M, B, E):
    cfg = wl.TraceConfig("g", E, N, M, 1, (N, N), (1, 1), "mix", dense_n=(N // 3, 2 * N))
    H = wl.make_dense_hist(cfg, seed=N + B).numpy()
    pos, npos, cost, cbb = sp.place_checkpoints_grid(torch.from_numpy(H).to(dev), M, B,
                                                     cost_by_budget=True)
    torch.cuda.synchronize()
    pos, npos, cost, cbb = np_(pos), np_(npos), np_(cost), np_(cbb)
    for e in range(E):
        rp, rc, rcbb = oracle.place_grid(H[e].astype(np.int64), M, B)
        assert npos[e] == len(rp) and pos[e, :len(rp)].tolist() == rp.tolist(), (e, pos[e], rp)
        assert (pos[e, len(rp):] == 0).all()
        assert cost[e] == rc and (cbb[e] == rcbb).all()
        assert oracle.expected_cost(H[e].astype(np.int64), rp) == rc


def test_grid_dp_sparse_lcp_histograms(dev):
    cfg = wl.scaled(wl.CONFIGS["W3"], 10)
    tr = wl.make_trace(cfg, seed=3)
    h, _ = oracle.lcp_hist(*(tr[k].numpy() for k in ("entry_tokens", "entry_off", "req_tokens",
                                                     "req_off", "req_entry")), cfg.N)
    for B in (64, 128):
        pos, npos, cost, _ = sp.place_checkpoints_grid(torch.from_numpy(h).to(dev), cfg.M, B)
        torch.cuda.synchronize()
        for e in range(10):
            rp, rc, _ = oracle.place_grid(h[e].astype(np.int64), cfg.M, B)
            assert np_(npos)[e] == len(rp) and np_(pos)[e, :len(rp)].tolist() == rp.tolist()
            assert np_(cost)[e] == rc


def test_grid_dp_f64(dev):
    N, M, B, E = 2048, 8, 64, 6
    cfg = wl.TraceConfig("g", E, N, M, 1, (N, N), (1, 1), "mix", dense_n=(3000, 9000))
    H = wl.make_dense_hist(cfg, seed=9).numpy().astype(np.int64)
    n = H.sum(1, keepdims=True)
    _, _, cost, _ = sp.place_checkpoints_grid(torch.from_numpy(H / n).to(dev), M, B)
    torch.cuda.synchronize()
    for e in range(E):
        _, rc, _ = oracle.place_grid(H[e], M, B)
        ref = rc / n[e, 0]
        assert abs(np_(cost)[e] - ref) <= 1e-12 * ref


def test_clip_parity_and_dominance(dev):
    cfg = wl.scaled(wl.CONFIGS["W4"], 24)
    H = wl.make_dense_hist(cfg, seed=4).to(dev)
    pos, npos, cost, _ = sp.place_checkpoints(H, 32)
    for B in (64, 128):
        cp, cn = sp.clip_to_blocks(pos, npos, B)
        gpos, gn, gcost, _ = sp.place_checkpoints_grid(H, 32, B)
        ccost, _ = sp.expected_recompute(H, cp.view(24, 1, 32), cn.view(24, 1), broadcast=False)
        torch.cuda.synchronize()
        P, K, CP, CN = np_(pos), np_(npos), np_(cp), np_(cn)
        for e in range(24):
            ref = oracle.clip_to_blocks(P[e, :K[e]], B)
            assert CN[e] == len(ref) and CP[e, :CN[e]].tolist() == ref.tolist()
            assert (CP[e, CN[e]:] == 0).all()
        # the exact block-restricted DP is never worse than post-hoc clipping
        assert (np_(gcost) <= np_(ccost)[:, 0]).all()
        assert (np_(gcost) >= np_(cost)).all()   # ... and never better than unrestricted
