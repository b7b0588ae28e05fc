"""Pins for the sampler variants of SURVEY 8(f) rank 2 in the CPU oracle (no GPU):
  * hop_time="root" (R#23): hop roots carry their layer-0 root's time ("others use the
    root's timestamp") -- against oracle/brute.py (a scan of the whole logical stream) and the
    no-leak invariant relative to the ROOT time;
  * uniform with replacement (R#24): against brute force, special cases (c = 0 -> nothing,
    c = 1 -> k copies of the only candidate) and the distribution of single draws (chi-square).
"""
import math

import numpy as np
import pytest

import oracle
from oracle import brute
from synth.tiny import random_graph, random_roots


def _compare(blocks, bf):
    for idx, (b, rows) in enumerate(zip(blocks, bf)):
        assert list(np.diff(b["offsets"])) == [len(r) for r in rows], f"block {idx}"
        flat = [x for r in rows for x in r]
        assert list(b["nbr"]) == [x[0] for x in flat]
        assert list(b["eid"]) == [x[1] for x in flat]
        np.testing.assert_array_equal(b["dt"].view(np.uint32), np.array([x[2] for x in flat], np.float32).view(np.uint32))


@pytest.mark.parametrize("hop_time,replacement", [("root", False), ("edge", True), ("root", True)])
def test_variants_match_brute_force(hop_time, replacement):
    rng = np.random.default_rng(11 + replacement + 2 * (hop_time == "root"))
    for case in range(80):
        n_nodes = int(rng.integers(1, 50))
        src, dst, ts, eid = random_graph(500 + case, n_nodes, int(rng.integers(0, 300)),
                                         integer_times=case % 3 != 0)
        roots, rts = random_roots(500 + case, n_nodes, int(rng.integers(1, 30)), integer_times=case % 3 != 0)
        L = 1 + case % 3
        fanouts = [int(rng.integers(1, 6)) for _ in range(L)]
        strategy = 1 if replacement else int(rng.integers(0, 2))
        S = int(rng.integers(1, 4))
        t_s = math.inf if S == 1 and case % 2 else float(rng.choice([1.0, 2.5, 7.0]))
        seed, base = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**40))
        add_rev = bool(case % 2)
        g = oracle.build(src, dst, ts, eid, n_nodes=n_nodes, add_reverse=add_rev)
        blocks = oracle.sample(g, roots, rts, fanouts=fanouts, strategy=strategy, n_snapshots=S, snapshot_len=t_s,
                               seed=seed, root_key_base=base, hop_time=hop_time, replacement=replacement)
        bf = brute.sample(src, dst, ts, eid, n_nodes=n_nodes, add_reverse=add_rev, roots=roots, root_ts=rts,
                          fanouts=fanouts, strategy=strategy, n_snapshots=S, snapshot_len=t_s, seed=seed,
                          root_key_base=base, hop_time=hop_time, replacement=replacement)
        _compare(blocks, bf)


def test_root_time_hops_are_earlier_than_the_root():
    """Every edge sampled at any layer is strictly earlier than its layer-0 root."""
    src, dst, ts, _ = random_graph(9, 60, 2000, integer_times=True, t_max=500)
    g = oracle.build(src, dst, ts, n_nodes=60, add_reverse=True)
    roots, rts = random_roots(9, 60, 200, integer_times=True, t_max=500)
    bl = oracle.sample(g, roots, rts, fanouts=[4, 3, 2], strategy=1, seed=5, hop_time="root")
    t = rts.astype(np.float32)
    for b in bl:
        cnt = np.diff(b["offsets"])
        t_edge = np.repeat(t, cnt) - b["dt"]
        assert np.all(b["dt"] > 0)
        assert np.all(t_edge < np.repeat(t, cnt))
        t = np.repeat(t, cnt)  # the next layer's roots carry the same root time


def test_with_replacement_special_cases():
    # one node 0 with c edges at times 0..c-1; roots at t = 100 (all candidates)
    for c, k in [(0, 3), (1, 5), (2, 7), (9, 4)]:
        src = np.zeros(c, np.int32)
        dst = np.ones(c, np.int32)
        g = oracle.build(src, dst, np.arange(c, dtype=np.float32), n_nodes=2, add_reverse=False)
        b = oracle.sample(g, np.zeros(50, np.int32), np.full(50, 100.0, np.float32), fanouts=[k], strategy=1,
                          seed=3, replacement=True)[0]
        cnt = np.diff(b["offsets"])
        assert np.all(cnt == (k if c else 0))
        if c:
            rows = b["eid"].reshape(50, k)
            assert np.all(np.diff(rows, axis=1) >= 0)       # ascending, duplicates allowed
            assert rows.min() >= 0 and rows.max() < c
            if c == 1:
                assert np.all(rows == 0)


def test_with_replacement_draws_uniform():
    """Single draws (k = 1) over many root keys are uniform over the c candidates (chi-square);
    with k = 6 > c = 5 duplicates occur (would be impossible without replacement)."""
    from scipy.stats import chisquare
    c = 13
    src = np.zeros(c, np.int32)
    dst = np.ones(c, np.int32)
    g = oracle.build(src, dst, np.arange(c, dtype=np.float32), n_nodes=2, add_reverse=False)
    n = 40000
    b = oracle.sample(g, np.zeros(n, np.int32), np.full(n, 1e6, np.float32), fanouts=[1], strategy=1, seed=21,
                      replacement=True)[0]
    assert chisquare(np.bincount(b["eid"], minlength=c)).pvalue > 1e-4
    g5 = oracle.build(np.zeros(5, np.int32), np.ones(5, np.int32), np.arange(5, dtype=np.float32), n_nodes=2,
                      add_reverse=False)
    b = oracle.sample(g5, np.zeros(100, np.int32), np.full(100, 1e6, np.float32), fanouts=[6], strategy=1, seed=2,
                      replacement=True)[0]
    rows = b["eid"].reshape(100, 6)
    assert np.all(np.diff(rows, axis=1) >= 0) and np.any(np.diff(rows, axis=1) == 0)


@pytest.mark.parametrize("hop_time", ["edge", "root"])
def test_dedup_matches_brute_force(hop_time):
    """R#27: with dedup the hop roots are the distinct (node, time) pairs; the brute force builds
    them with a set over its own scan of the logical stream."""
    rng = np.random.default_rng(77 + (hop_time == "root"))
    for case in range(60):
        n_nodes = int(rng.integers(1, 30))
        src, dst, ts, eid = random_graph(700 + case, n_nodes, int(rng.integers(0, 300)), integer_times=True,
                                         t_max=8.0)  # few distinct times: many duplicate pairs
        roots, rts = random_roots(700 + case, n_nodes, int(rng.integers(1, 30)), integer_times=True, t_max=8.0)
        L = 1 + case % 3
        fanouts = [int(rng.integers(1, 6)) for _ in range(L)]
        strategy = int(rng.integers(0, 2))
        S = 1 if L > 1 else int(rng.integers(1, 4))
        t_s = math.inf if S == 1 else 2.5
        seed, base = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**40))
        g = oracle.build(src, dst, ts, eid, n_nodes=n_nodes, add_reverse=bool(case % 2))
        blocks = oracle.sample(g, roots, rts, fanouts=fanouts, strategy=strategy, n_snapshots=S, snapshot_len=t_s,
                               seed=seed, root_key_base=base, hop_time=hop_time, dedup=True)
        bf = brute.sample(src, dst, ts, eid, n_nodes=n_nodes, add_reverse=bool(case % 2), roots=roots, root_ts=rts,
                          fanouts=fanouts, strategy=strategy, n_snapshots=S, snapshot_len=t_s, seed=seed,
                          root_key_base=base, hop_time=hop_time, dedup=True)
        _compare(blocks, bf)
        for b in blocks:  # src_index maps every output to its (node, time) pair
            assert np.array_equal(b["uniq_node"][b["src_index"]], b["nbr"])
            assert len(set(zip(b["uniq_node"].tolist(), b["uniq_ts"].view(np.uint32).tolist()))) == len(b["uniq_node"])


def _mask(rng, n_edges, frac):
    bits = rng.random(max(n_edges, 1)) < frac
    words = np.zeros((len(bits) + 31) // 32, dtype=np.uint32)
    for e in np.nonzero(bits)[0]:
        words[e >> 5] |= np.uint32(1) << np.uint32(e & 31)
    return words


@pytest.mark.parametrize("strategy,replacement", [(0, False), (1, False), (1, True)])
def test_edge_validity_matches_brute_force(strategy, replacement):
    """R#28: invalid edges are skipped; vs the brute-force scan with the same mask."""
    rng = np.random.default_rng(300 + strategy + 2 * replacement)
    for case in range(60):
        n_nodes = int(rng.integers(1, 40))
        n_edges = int(rng.integers(0, 300))
        src, dst, ts, eid = random_graph(1100 + case, n_nodes, n_edges, integer_times=case % 3 != 0)
        roots, rts = random_roots(1100 + case, n_nodes, int(rng.integers(1, 30)), integer_times=case % 3 != 0)
        L = 1 + case % 2
        fanouts = [int(rng.integers(1, 6)) for _ in range(L)]
        S = int(rng.integers(1, 4))
        t_s = math.inf if S == 1 and case % 2 else 2.5
        seed, base = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**40))
        valid = _mask(rng, n_edges, float(rng.choice([0.0, 0.3, 0.8, 1.0])))
        g = oracle.build(src, dst, ts, eid, n_nodes=n_nodes, add_reverse=bool(case % 2))
        blocks = oracle.sample(g, roots, rts, fanouts=fanouts, strategy=strategy, n_snapshots=S, snapshot_len=t_s,
                               seed=seed, root_key_base=base, replacement=replacement, edge_valid=valid)
        bf = brute.sample(src, dst, ts, eid, n_nodes=n_nodes, add_reverse=bool(case % 2), roots=roots, root_ts=rts,
                          fanouts=fanouts, strategy=strategy, n_snapshots=S, snapshot_len=t_s, seed=seed,
                          root_key_base=base, replacement=replacement, edge_valid=valid)
        _compare(blocks, bf)


def test_edge_validity_all_valid_and_none_valid():
    src, dst, ts, _ = random_graph(4, 30, 400)
    roots, rts = random_roots(4, 30, 50)
    g = oracle.build(src, dst, ts, n_nodes=30, add_reverse=True)
    kw = dict(fanouts=[5, 3], strategy=1, seed=8)
    plain = oracle.sample(g, roots, rts, **kw)
    full = oracle.sample(g, roots, rts, edge_valid=np.full(13, 0xFFFFFFFF, np.uint32), **kw)
    for a, b in zip(plain, full):
        assert np.array_equal(a["nbr"], b["nbr"]) and np.array_equal(a["offsets"], b["offsets"])
    none = oracle.sample(g, roots, rts, edge_valid=np.zeros(13, np.uint32), **kw)
    assert all(len(b["nbr"]) == 0 for b in none)
