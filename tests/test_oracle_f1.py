"""Pins for the f1 (block-aware placement) part of the oracle: SPEC's worked examples for
clipping / sqrt / logarithmic schedules (Table 1), brute force over grid
subsets for the block-restricted DP, B = 1 reducing to the unrestricted DP, and the SPEC
invariants "clipping never increases the reusable depth" and "block-restricted
DP cost <= clip(DP) cost"."""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from paper_2605_05219_b200 import workload as wl

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("ex", GOLD["clip_to_blocks"], ids=lambda e: e["cite"][:12])
def test_golden_clip(ex):
    assert oracle.clip_to_blocks(ex["C"], ex["B"]).tolist() == ex["out"]


@pytest.mark.parametrize("ex", GOLD["sqrt_placement"], ids=lambda e: e["cite"][:12])
def test_golden_sqrt(ex):
    assert oracle.sqrt_positions(ex["N"]).tolist() == ex["out"]


@pytest.mark.parametrize("ex", GOLD["logarithmic_placement"], ids=lambda e: e["cite"][:12])
def test_golden_log(ex):
    assert oracle.log_positions(ex["N"], ex["M"]).tolist() == ex["out"]


def test_log_dedup_and_growth():
    """N=4, M=3 -> strictly increasing, size <= 3; gaps grow toward the end."""
    p = oracle.log_positions(4, 3)
    assert len(p) <= 3 and (np.diff(p) > 0).all()
    p = oracle.log_positions(32768, 12)
    g = np.diff(np.concatenate([[0], p]))
    assert (np.diff(g) >= -1).all() and p[-1] == 32768


def _grid_brute(c, M, B):
    N = len(c) - 1
    grid = list(range(B, N + 1, B))
    best = None
    for k in range(0, min(M, len(grid)) + 1):
        for C in itertools.combinations(grid, k):
            v = oracle.expected_cost(c, np.asarray(C, np.int32))
            key = (v, tuple(sorted(C, reverse=True)))
            if best is None or key < best:
                best = key
    return sorted(best[1]), best[0]


def test_grid_dp_equals_brute_force():
    for key in range(250):
        N = 3 + key % 28
        B = 1 + key % 6
        M = key % 5
        M = min(M, N)
        c = wl.random_small_hist(13, N, max_count=6, zero_frac=0.4, key=key).numpy()
        pos, cost, _ = oracle.place_grid(c, M, B)
        bpos, bcost = _grid_brute(c, M, B)
        assert cost == bcost, (key, N, B, M)
        assert pos.tolist() == bpos, (key, pos, bpos)
        assert all(p % B == 0 for p in pos)


def test_grid_b1_is_unrestricted():
    for key in range(40):
        N = 5 + key * 3
        c = wl.random_small_hist(14, N, max_count=9, zero_frac=0.3, key=key).numpy()
        for M in (0, 1, 4):
            p1, v1, cb1 = oracle.place_grid(c, M, 1)
            p2, v2, cb2 = oracle.place(c, M, "naive")
            assert v1 == v2 and p1.tolist() == p2.tolist() and (cb1 == cb2).all()


def test_clip_properties_and_grid_dominance():
    rng = np.random.default_rng(4)
    for _ in range(300):
        N = int(rng.integers(10, 400))
        B = int(rng.integers(1, 70))
        k = int(rng.integers(0, min(N, 12) + 1))
        C = np.sort(rng.choice(np.arange(1, N + 1), size=k, replace=False)).astype(np.int32)
        cl = oracle.clip_to_blocks(C, B)
        assert all(p % B == 0 and p >= B for p in cl) and len(cl) <= len(C)
        for t in rng.integers(1, N + 1, size=10):
            # feasibility (a clipped state never lies above the depth it serves).  SPEC's
            # stronger claim l(t; clip(C)) <= l(t; C) is false -- see
            # test_spec_clip_monotonicity_counterexample and DESIGN.md reading R14
            l1 = max([0] + [p for p in cl if p <= t])
            assert l1 <= t
            assert all(p in cl for p in ((q // B) * B for q in C) if p > 0)
    for key in range(40):   # block-restricted DP <= post-hoc clipping of the DP
        N = 40 + key * 7
        c = wl.random_small_hist(15, N, max_count=9, zero_frac=0.5, key=key).numpy()
        for B in (4, 16):
            for M in (1, 3, 6):
                pos, _, _ = oracle.place(c, M, "cht")
                _, gcost, _ = oracle.place_grid(c, M, B)
                assert gcost <= oracle.expected_cost(c, oracle.clip_to_blocks(pos, B))


def test_spec_clip_monotonicity_counterexample():
    """S:241/S:567 claim clipping never increases l(t;C); flooring can move a checkpoint below
    a depth it used to exceed: C = {184, 200}, B = 99, t = 199."""
    C = np.array([184, 200], np.int32)
    cl = oracle.clip_to_blocks(C, 99)
    assert cl.tolist() == [99, 198]
    l_clip = max([0] + [p for p in cl if p <= 199])
    l_orig = max([0] + [p for p in C if p <= 199])
    assert (l_clip, l_orig) == (198, 184)
