"""GPU parity for f4: longest-prefix search over all cached entries,
sp_prefix_index_build + sp_match_longest_prefix against the oracle's brute force -- bit-exact
entry and depth, including the most-recent tie rule."""
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
    sp.lib()
    return torch.device("cuda:0")


def csr(seqs):
    off = np.zeros(len(seqs) + 1, np.int64)
    off[1:] = np.cumsum([len(s) for s in seqs])
    tok = np.concatenate([np.asarray(s, np.int32) for s in seqs]) if off[-1] else np.zeros(0, np.int32)
    return tok, off


def gpu_match(et, eo, rt, ro, dev, insertion=None):
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    idx = sp.PrefixIndex(T(et), T(eo), None if insertion is None else T(insertion))
    me, md = idx.match(T(rt), T(ro))
    torch.cuda.synchronize()
    return me.cpu().numpy(), md.cpu().numpy()


def check(et, eo, rt, ro, dev, insertion=None):
    me, md = gpu_match(et, eo, rt, ro, dev, insertion)
    re_, rd = oracle.match_longest_prefix(et, eo, rt, ro, insertion)
    assert (md == rd).all(), np.nonzero(md != rd)
    assert (me == re_).all(), np.nonzero(me != re_)


def test_spec_examples(dev):
    A, B, C, D, X, Y, Z = range(1, 8)
    check(*csr([[A, B, C, X], [A, B, Y, Z]]), *csr([[A, B, C, D], [A, B, Y, Z], [Z], [A]]), dev)


def test_empty_cache(dev):
    me, md = gpu_match(*csr([]), *csr([[1, 2], [3]]), dev)
    assert me.tolist() == [-1, -1] and md.tolist() == [0, 0]


@pytest.mark.parametrize("alpha,seed", [(2, 0), (3, 1), (50, 2)])
def test_random_shared_prefixes(dev, alpha, seed):
    """Small alphabets: many entries share long prefixes, duplicates and prefix-of-prefix
    entries, many ties (resolved by entry index, then by a random insertion order)."""
    rng = np.random.default_rng(seed)
    base = rng.integers(0, alpha, 300)
    ents = [np.concatenate([base[:rng.integers(0, 300)], rng.integers(0, alpha, rng.integers(0, 40))])
            for _ in range(257)]
    ents += [ents[3], ents[3], base[:10]]
    reqs = [np.concatenate([base[:rng.integers(0, 300)], rng.integers(0, alpha, rng.integers(0, 50))])
            for _ in range(1000)] + [ents[3], [], base[:10], base]
    et, eo = csr(ents)
    rt, ro = csr(reqs)
    check(et, eo, rt, ro, dev)
    check(et, eo, rt, ro, dev, insertion=rng.permutation(len(ents)).astype(np.int64) // 2)


def test_w2_trace_matches_own_entry(dev):
    """W2-shaped trace (S:477 construction: request = entry prefix + disjoint suffix): the search
    over all 200 entries finds the request's own entry at the drawn depth (misses: none)."""
    cfg = wl.scaled(wl.CONFIGS["W2"], 200)
    tr = wl.make_trace(cfg, seed=4)
    et, eo = tr["entry_tokens"].numpy(), tr["entry_off"].numpy()
    rt, ro = tr["req_tokens"].numpy(), tr["req_off"].numpy()
    check(et, eo, rt, ro, dev)
    me, md = gpu_match(et, eo, rt, ro, dev)
    _, lcp = oracle.lcp_hist(et, eo, rt, ro, tr["req_entry"].numpy(), cfg.N, n_entries=200)
    hit = md > 0
    assert (me[hit] == tr["req_entry"].numpy()[hit]).all()
    assert (np.minimum(md, cfg.N) == lcp).all()
