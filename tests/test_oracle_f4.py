"""Oracle pins for f4: longest-prefix match against all cached entries (SPEC
match_longest_prefix S:375-383) -- SPEC's worked examples, the single-entry case against the
oracle's a1 LCP loop, and brute-force properties on random caches with shared prefixes."""
import numpy as np

import oracle


def csr(seqs):
    off = np.zeros(len(seqs) + 1, np.int64)
    off[1:] = np.cumsum([len(s) for s in seqs])
    tok = np.concatenate([np.asarray(s, np.int32) for s in seqs]) if off[-1] else np.zeros(0, np.int32)
    return tok, off


def test_spec_examples():
    A, B, C, D, X, Y, Z = range(1, 8)
    et, eo = csr([])                                                   # S:380 empty cache
    me, md = oracle.match_longest_prefix(et, eo, *csr([[A, B]]))
    assert me.tolist() == [-1] and md.tolist() == [0]
    et, eo = csr([[A, B, C, X], [A, B, Y, Z]])
    me, md = oracle.match_longest_prefix(et, eo, *csr([[A, B, C, D]]))
    assert me.tolist() == [0] and md.tolist() == [3]
    me, md = oracle.match_longest_prefix(et, eo, *csr([[A, B, Y, Z]])) # S:381 identical
    assert me.tolist() == [1] and md.tolist() == [4]


def test_ties_most_recent_insertion():
    et, eo = csr([[1, 2, 3], [1, 2, 9], [1, 2, 8]])
    rt, ro = csr([[1, 2, 7], [5]])
    me, md = oracle.match_longest_prefix(et, eo, rt, ro)
    assert me.tolist() == [2, -1] and md.tolist() == [2, 0]
    me, md = oracle.match_longest_prefix(et, eo, rt, ro, insertion=np.array([5, 9, 1]))
    assert me.tolist() == [1, -1]


def test_single_entry_equals_a1_lcp_loop():
    rng = np.random.default_rng(0)
    ent = rng.integers(0, 4, 50)
    reqs = [np.concatenate([ent[:k], rng.integers(0, 4, 5)]) for k in range(0, 50, 3)]
    et, eo = csr([ent])
    rt, ro = csr(reqs)
    me, md = oracle.match_longest_prefix(et, eo, rt, ro)
    h, lcp = oracle.lcp_hist(et, eo, rt, ro, np.zeros(len(reqs), np.int32), 100)
    assert (md == lcp).all() and (me == np.where(lcp > 0, 0, -1)).all()


def test_random_caches_properties():
    """Small alphabet, shared prefixes: the match has the maximum LCP over all entries (checked
    entry by entry with the a1 loop), and no more recent entry reaches it."""
    rng = np.random.default_rng(1)
    base = rng.integers(0, 3, 40)
    ents = [np.concatenate([base[:rng.integers(0, 40)], rng.integers(0, 3, rng.integers(0, 20))])
            for _ in range(30)]
    reqs = [np.concatenate([base[:rng.integers(0, 40)], rng.integers(0, 3, 10)]) for _ in range(60)]
    et, eo = csr(ents)
    rt, ro = csr(reqs)
    me, md = oracle.match_longest_prefix(et, eo, rt, ro)
    for r in range(len(reqs)):
        lc = []
        for e in range(len(ents)):
            _, l = oracle.lcp_hist(*csr([ents[e]]), *csr([reqs[r]]), np.zeros(1, np.int32), 1000)
            lc.append(int(l[0]))
        mx = max(lc)
        assert md[r] == mx
        if mx == 0:
            assert me[r] == -1
        else:
            assert lc[me[r]] == mx and all(l < mx for l in lc[me[r] + 1:])
