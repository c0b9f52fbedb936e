"""GPU parity for f2 (Thm 4's exponentially weighted histogram): the batched device
estimator (sp_gamma_observe / sp_gamma_snapshot) against the oracle's definitional formula,
and the estimator -> fp64 DP path (the paper's method) against the oracle's fp64 DP."""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_05219_b200 import sp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2605_05219_b200 import build
    build.build()
    sp.lib()
    return torch.device("cuda:0")


def streams(E, N, lens, seed):
    rng = np.random.default_rng(seed)
    out = []
    for e in range(E):
        n = int(lens[e])
        # a drifting law: depths from a moving window, plus misses and depths beyond N
        centre = (np.arange(n) * 7 // max(n, 1) + e) % N
        d = np.clip(centre + rng.integers(-30, 31, n), -2, N + 5)
        d[rng.random(n) < 0.05] = 0
        out.append(d.astype(np.int32))
    return out


def run_batches(est, per_entry, batches, dev):
    """Feed each entry's stream in `batches` consecutive CSR batches."""
    E = len(per_entry)
    cuts = [np.linspace(0, len(d), batches + 1).astype(int) for d in per_entry]
    for b in range(batches):
        parts = [per_entry[e][cuts[e][b]:cuts[e][b + 1]] for e in range(E)]
        off = np.zeros(E + 1, np.int64)
        off[1:] = np.cumsum([len(x) for x in parts])
        dep = np.concatenate(parts) if off[-1] else np.zeros(0, np.int32)
        est.observe(torch.from_numpy(off).to(dev), torch.from_numpy(dep).to(dev))


@pytest.mark.parametrize("g,batches", [(0.99, 1), (0.99, 7), (0.5, 3), (0.9, 5), (1.0, 4)])
def test_gamma_snapshot_vs_definition(dev, g, batches):
    E, N = 12, 300
    lens = [1, 2, 10, 100, 1000, 9000, 20000, 0, 5, 3000, 64, 777]   # > 2^64 exponent ranges
    per = streams(E, N, lens, seed=int(g * 100) + batches)
    est = sp.GammaEstimator(E, N, g, device=dev)
    run_batches(est, per, batches, dev)
    p = est.snapshot().cpu().numpy()
    hits = np.array([(d >= 1).sum() for d in per])             # t counts hits (reading R15)
    assert (est.t.cpu().numpy() == hits).all()
    for e in range(E):
        if hits[e] == 0:
            assert (p[e] == 0).all()
            continue
        ref = oracle.gamma_hist(per[e], N, g)
        assert np.allclose(p[e], ref, rtol=1e-12, atol=1e-15), (e, np.abs(p[e] - ref).max())
        assert abs(p[e].sum() - 1) < 1e-12


def test_gamma_estimator_feeds_fp64_dp(dev):
    """The paper's method: DP on the g = 0.99 estimate.  The device DP runs on the
    unnormalised W (scale-invariant); its placement is scored under the oracle's p_t and must be
    optimal to 1e-12 relative (the fp64 reading R10)."""
    E, N, M = 6, 500, 12
    per = streams(E, N, [400, 1000, 3000, 50, 2000, 7000], seed=3)
    est = sp.GammaEstimator(E, N, 0.99, device=dev)
    run_batches(est, per, 4, dev)
    pos, npos, cost, _ = sp.place_checkpoints(est.W.contiguous(), M)
    torch.cuda.synchronize()
    pos, npos = pos.cpu().numpy(), npos.cpu().numpy()
    for e in range(E):
        ref = oracle.gamma_hist(per[e], N, 0.99)
        D, _ = oracle.dp_f64(ref, M)
        best = D[M][N]
        got = oracle.expected_cost_f64(ref, pos[e, :npos[e]])
        assert got <= best * (1 + 1e-12) + 1e-15, (e, got, best)


def test_gamma_errors(dev):
    est = sp.GammaEstimator(2, 10, 0.9, device=dev)
    with pytest.raises(sp.SPError):
        sp.gamma_observe(est.W, est.t, est.tau, torch.zeros(3, dtype=torch.int64, device=dev),
                         torch.zeros(1, dtype=torch.int32, device=dev), 1.5)
