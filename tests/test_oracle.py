"""Pins for the CPU oracle (oracle/tgl_oracle.c) against things other than itself.

Every test here runs without a GPU.  Pins (SURVEY 8(c) "What pins each part"):
  * Philox4x32-10 known-answer vectors (tests/golden/philox_kat.json)
  * the paper's Fig. 3 hand example and the add_reverse tie example
  * numpy stable argsort for the T-CSR build (a library sort vs a counting sort)
  * oracle/brute.py: a scan of the whole logical edge stream, on 200 random graphs
  * invariants: no leak, count = min(k, c), ascending output, snapshot
    windows partition [t - S ts, t), dt > 0 under gradual underflow
  * the uniform draw: exhaustive subset frequencies and per-slot inclusion k/c
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import brute
from synth.tiny import random_graph, random_roots


def _hex(xs):
    return [int(x, 16) for x in xs]


# --------------------------------------------------------------------------- Philox
def test_philox_known_answers(golden_dir):
    kat = json.load(open(os.path.join(golden_dir, "philox_kat.json")))
    for v in kat["vectors"]:
        want = _hex(v["out"])
        assert list(oracle.philox4x32_10(_hex(v["ctr"]), _hex(v["key"]))) == want
        assert brute.philox(_hex(v["ctr"]), _hex(v["key"])) == want


def test_philox_two_implementations_agree_random():
    rng = np.random.default_rng(1)
    for _ in range(200):
        ctr = rng.integers(0, 2**32, size=4, dtype=np.uint64)
        key = rng.integers(0, 2**32, size=2, dtype=np.uint64)
        assert list(oracle.philox4x32_10(ctr, key)) == brute.philox(ctr, key)


# --------------------------------------------------------------------------- golden examples
def _run_case(g, case, n_nodes):
    ts_len = math.inf if case["snapshot_len"] == "inf" else float(case["snapshot_len"])
    return oracle.sample(g, [case["root"]], [case["t"]], fanouts=case["fanouts"],
                         strategy=case["strategy"], n_snapshots=case["n_snapshots"],
                         snapshot_len=ts_len, seed=0, root_key_base=0)


@pytest.mark.parametrize("name", ["fig3.json", "ties.json", "r3_hops.json"])
def test_golden_examples(golden_dir, name):
    gd = json.load(open(os.path.join(golden_dir, name)))
    e = gd["edges"]
    g = oracle.build(e["src"], e["dst"], np.float32(e["ts"]), n_nodes=gd["n_nodes"],
                     add_reverse=bool(gd["add_reverse"]))
    if "expect_tcsr" in gd:
        for key, want in gd["expect_tcsr"].items():
            np.testing.assert_array_equal(g[key], np.asarray(want, dtype=g[key].dtype))
    if "expect_node0" in gd:
        lo, hi = g["indptr"][0], g["indptr"][1]
        assert list(g["nbr"][lo:hi]) == gd["expect_node0"]["nbr"]
        assert list(g["eid"][lo:hi]) == gd["expect_node0"]["eid"]
    for case in gd["cases"]:
        blocks = _run_case(g, case, gd["n_nodes"])
        assert len(blocks) == len(case["blocks"]), case["what"]
        for b, want in zip(blocks, case["blocks"]):
            assert list(b["nbr"]) == want["nbr"], case["what"]
            assert list(b["eid"]) == want["eid"], case["what"]
            assert [float(x) for x in b["dt"]] == want["dt"], case["what"]
            assert list(b["offsets"]) == [0, len(want["nbr"])], case["what"]


# --------------------------------------------------------------------------- build
@pytest.mark.parametrize("add_reverse", [False, True])
def test_build_matches_stable_argsort(add_reverse):
    for seed in range(40):
        n_nodes = [1, 2, 7, 33, 200][seed % 5]
        n_edges = [0, 1, 5, 300, 2000][(seed // 5) % 5]
        src, dst, ts, eid = random_graph(seed, n_nodes, n_edges, with_eid=bool(seed % 2))
        g = oracle.build(src, dst, ts, eid, n_nodes=n_nodes, add_reverse=add_reverse)
        ref = brute.tcsr(src, dst, ts, eid, n_nodes=n_nodes, add_reverse=add_reverse)
        for key in ("indptr", "nbr", "ts", "eid"):
            np.testing.assert_array_equal(g[key], ref[key])
        # invariants: sum of degrees = E_s, lists non-decreasing in time
        assert g["indptr"][-1] == n_edges * (2 if add_reverse else 1)
        for v in range(n_nodes):
            seg = g["ts"][g["indptr"][v]:g["indptr"][v + 1]]
            assert np.all(np.diff(seg) >= 0)


def test_build_empty_graph_and_isolated_nodes():
    g = oracle.build([], [], np.zeros(0, np.float32), n_nodes=3, add_reverse=False)
    assert list(g["indptr"]) == [0, 0, 0, 0]
    g = oracle.build([0], [2], np.float32([1.0]), n_nodes=4, add_reverse=True)
    assert list(g["indptr"]) == [0, 1, 1, 2, 2]                   # nodes 1, 3 isolated


@pytest.mark.parametrize("src,dst,ts,code", [
    ([0, 5], [1, 1], [0.0, 1.0], oracle.ERANGE),
    ([0, -1], [1, 1], [0.0, 1.0], oracle.ERANGE),
    ([0, 1], [1, 1], [-1.0, 1.0], oracle.EINVAL),
    ([0, 1], [1, 1], [0.0, float("nan")], oracle.EINVAL),
    ([0, 1], [1, 1], [0.0, float("inf")], oracle.EINVAL),
    ([0, 1], [1, 1], [2.0, 1.0], oracle.EUNSORTED),
])
def test_build_validation(src, dst, ts, code):
    with pytest.raises(oracle.OracleError) as ei:
        oracle.build(src, dst, np.float32(ts), n_nodes=3, add_reverse=False)
    assert ei.value.code == code


def test_restricted_build_equals_full_on_kept_nodes():
    src, dst, ts, eid = random_graph(5, 50, 3000, with_eid=True)
    full = oracle.build(src, dst, ts, eid, n_nodes=50, add_reverse=True)
    keep = np.zeros(50, np.uint8)
    keep[[0, 3, 7, 49]] = 1

    def chunks():
        for a in range(0, 3000, 700):
            yield src[a:a + 700], dst[a:a + 700], ts[a:a + 700], eid[a:a + 700], a

    part = oracle.build_restricted(chunks, n_nodes=50, add_reverse=True, keep=keep)
    for v in range(50):
        fl = slice(full["indptr"][v], full["indptr"][v + 1])
        pl = slice(part["indptr"][v], part["indptr"][v + 1])
        if keep[v]:
            for key in ("nbr", "ts", "eid"):
                np.testing.assert_array_equal(part[key][pl], full[key][fl])
        else:
            assert pl.stop == pl.start
    # chunked default eid (None) = global input index
    def chunks2():
        for a in range(0, 3000, 700):
            yield src[a:a + 700], dst[a:a + 700], ts[a:a + 700], None, a
    part2 = oracle.build_restricted(chunks2, n_nodes=50, add_reverse=False, keep=keep)
    full2 = oracle.build(src, dst, ts, None, n_nodes=50, add_reverse=False)
    for v in np.nonzero(keep)[0]:
        fl = slice(full2["indptr"][v], full2["indptr"][v + 1])
        pl = slice(part2["indptr"][v], part2["indptr"][v + 1])
        np.testing.assert_array_equal(part2["eid"][pl], full2["eid"][fl])


# --------------------------------------------------------------------------- sampler vs brute force
def _compare_to_brute(blocks, bf, fanouts, S, check_children=True):
    for idx, (b, rows) in enumerate(zip(blocks, bf)):
        counts = np.diff(b["offsets"])
        assert list(counts) == [len(r) for r in rows], f"block {idx}"
        flat = [x for r in rows for x in r]
        assert list(b["nbr"]) == [x[0] for x in flat]
        assert list(b["eid"]) == [x[1] for x in flat]
        np.testing.assert_array_equal(b["dt"].view(np.uint32),
                                      np.array([x[2] for x in flat], np.float32).view(np.uint32))
        if "ts_edge" in b:
            np.testing.assert_array_equal(b["ts_edge"], np.array([x[3] for x in flat], np.float32))


def test_sampler_matches_brute_force_200_graphs():
    """SPEC acceptance #1 analogue: 200 random graphs, every block bit-identical."""
    rng = np.random.default_rng(2024)
    for case in range(200):
        n_nodes = int(rng.integers(1, 60))
        n_edges = int(rng.integers(0, 400))
        add_rev = bool(case % 2)
        integer_times = case % 3 != 0
        src, dst, ts, eid = random_graph(case, n_nodes, n_edges, with_eid=bool(case % 5 == 0),
                                         integer_times=integer_times)
        roots, rts = random_roots(case, n_nodes, int(rng.integers(1, 40)), integer_times=integer_times)
        L = 1 + case % 2
        fanouts = [int(rng.integers(1, 6)) for _ in range(L)]
        strategy = int(rng.integers(0, 2))
        S = int(rng.integers(1, 4))
        t_s = math.inf if S == 1 and case % 4 else float(rng.choice([1.0, 2.5, 7.0]))
        seed = int(rng.integers(0, 2**63))
        base = int(rng.integers(0, 2**40))
        g = oracle.build(src, dst, ts, eid, n_nodes=n_nodes, add_reverse=add_rev)
        blocks = oracle.sample(g, roots, rts, fanouts=fanouts, strategy=strategy, n_snapshots=S,
                               snapshot_len=t_s, seed=seed, root_key_base=base)
        bf = brute.sample(src, dst, ts, eid, n_nodes=n_nodes, add_reverse=add_rev, roots=roots,
                          root_ts=rts, fanouts=fanouts, strategy=strategy, n_snapshots=S,
                          snapshot_len=t_s, seed=seed, root_key_base=base)
        _compare_to_brute(blocks, bf, fanouts, S)


def test_invariants_no_leak_counts_partition():
    src, dst, ts, _ = random_graph(11, 40, 3000, integer_times=True)
    g = oracle.build(src, dst, ts, n_nodes=40, add_reverse=True)
    roots, rts = random_roots(11, 40, 300)
    S, t_s, k = 3, 4.0, 1000
    blocks = oracle.sample(g, roots, rts, fanouts=[k], strategy=0, n_snapshots=S, snapshot_len=t_s)
    # the S windows are disjoint and their union is [t - S*ts, t)
    union = oracle.sample(g, roots, rts, fanouts=[k], strategy=0, n_snapshots=1, snapshot_len=S * t_s)
    for i in range(len(roots)):
        parts = []
        for s in range(S):
            b = blocks[s]
            lo, hi = b["offsets"][i], b["offsets"][i + 1]
            parts.extend(zip(b["eid"][lo:hi], b["dt"][lo:hi]))
            # every edge strictly earlier than the root and inside window s
            assert np.all(b["dt"][lo:hi] > 0)
            assert np.all(b["dt"][lo:hi] <= (s + 1) * t_s)
        u = union[0]
        lo, hi = u["offsets"][i], u["offsets"][i + 1]
        assert sorted(parts) == sorted(zip(u["eid"][lo:hi], u["dt"][lo:hi]))


def test_multilayer_chain_strictly_decreasing_time():
    src, dst, ts, _ = random_graph(3, 30, 2000, integer_times=False)
    g = oracle.build(src, dst, ts, n_nodes=30, add_reverse=True)
    roots, rts = random_roots(3, 30, 50, integer_times=False)
    blocks = oracle.sample(g, roots, rts, fanouts=[4, 3], strategy=1, seed=9)
    b0, b1 = blocks
    # layer-1 roots are layer-0 outputs element for element (Alg. 1)
    assert len(b1["offsets"]) == len(b0["nbr"]) + 1
    for p in range(len(b0["nbr"])):
        lo, hi = b1["offsets"][p], b1["offsets"][p + 1]
        assert np.all(b1["dt"][lo:hi] > 0)                       # t_edge(1) < t_edge(0)
    for i in range(len(roots)):
        lo, hi = b0["offsets"][i], b0["offsets"][i + 1]
        np.testing.assert_array_equal(np.float32(rts[i]) - b0["ts_edge"][lo:hi], b0["dt"][lo:hi])
        assert np.all(b0["ts_edge"][lo:hi] < rts[i])


def test_dt_positive_under_gradual_underflow():
    tiny = np.float32(1.4e-45)                                  # smallest subnormal
    src, dst = [0, 0], [1, 2]
    ts = np.array([0.0, tiny], np.float32)
    g = oracle.build(src, dst, ts, n_nodes=3, add_reverse=False)
    t = np.float32(2 * tiny)
    b = oracle.sample(g, [0], [t], fanouts=[5], strategy=0)[0]
    assert list(b["nbr"]) == [1, 2]
    assert b["dt"][1] == tiny and b["dt"][1] > 0                 # FTZ would give 0


def test_bad_roots_give_zero_count_and_error():
    g = oracle.build([0], [1], np.float32([1.0]), n_nodes=2, add_reverse=True)
    b = oracle.sample_block(g, [5, 0, 0], np.float32([9, float("nan"), 9]), np.zeros(3, np.uint64), None,
                            layer=0, snapshot=0, snapshot_len=math.inf, k=3, strategy=0, seed=0,
                            want_children=False)
    assert list(b["offsets"]) == [0, 0, 0, 1]
    assert b["err"] != 0


# --------------------------------------------------------------------------- uniform distribution
def test_uniform_exhaustive_subset_frequencies():
    """For c <= 6, k <= 3, every k-subset appears with frequency 1/C(c,k) (chi-square)."""
    from itertools import combinations
    from scipy.stats import chisquare
    n_keys = 20000
    for c in range(2, 7):
        for k in range(1, min(3, c - 1) + 1):
            # one node with c edges, many roots (distinct keys) at a time after all of them
            src = np.zeros(c, np.int32)
            dst = np.arange(c, dtype=np.int32) % 2
            g = oracle.build(src, dst, np.arange(c, dtype=np.float32), n_nodes=2, add_reverse=False)
            b = oracle.sample(g, np.zeros(n_keys, np.int32), np.full(n_keys, 100.0, np.float32),
                              fanouts=[k], strategy=1, seed=12345, root_key_base=77)[0]
            subsets = list(combinations(range(c), k))
            index = {s: j for j, s in enumerate(subsets)}
            counts = np.zeros(len(subsets))
            eids = b["eid"].reshape(n_keys, k)
            for row in eids:
                counts[index[tuple(row)]] += 1
            p = chisquare(counts).pvalue
            assert p > 1e-4, (c, k, counts)


def test_uniform_inclusion_frequency():
    from scipy.stats import chisquare
    c, k, n_keys = 40, 10, 20000
    src = np.zeros(c, np.int32)
    dst = np.ones(c, np.int32)
    g = oracle.build(src, dst, np.arange(c, dtype=np.float32), n_nodes=2, add_reverse=False)
    b = oracle.sample(g, np.zeros(n_keys, np.int32), np.full(n_keys, 1e6, np.float32),
                      fanouts=[k], strategy=1, seed=99)[0]
    counts = np.bincount(b["eid"], minlength=c)
    assert counts.sum() == n_keys * k
    assert chisquare(counts).pvalue > 1e-4
    rows = b["eid"].reshape(n_keys, k)
    assert np.all(np.diff(rows, axis=1) > 0)                     # distinct, ascending


# --------------------------------------------------------------------------- gather
def test_gather_bytes():
    rng = np.random.default_rng(0)
    table = rng.standard_normal((17, 5)).astype(np.float32)
    ids = np.array([3, -1, 16, 0, 3], np.int32)
    out, err = oracle.gather(ids, table)
    assert err == 0
    want = np.zeros((5, 5), np.float32)
    for i, j in enumerate(ids):
        if j >= 0:
            want[i] = table[j]
    np.testing.assert_array_equal(out.view(np.uint32), want.view(np.uint32))
    out, err = oracle.gather(np.array([17], np.int32), table)
    assert err != 0 and not out.any()


def test_fnv1a64_published_vectors():
    """The digest used for per-batch parity against the FNV-1a-64 test vectors
    published with the algorithm (Fowler/Noll/Vo): "" / "a" / "foobar"."""
    assert oracle.fnv1a64(b"") == 0xcbf29ce484222325
    assert oracle.fnv1a64(b"a") == 0xaf63dc4c8601ec8c
    assert oracle.fnv1a64(b"foobar") == 0x85944171f73967e8
    # continuation == one pass over the concatenation
    assert oracle.fnv1a64(b"bar", oracle.fnv1a64(b"foo")) == oracle.fnv1a64(b"foobar")


def test_block_digest_byte_order():
    """oracle.block_digest hashes rebased int64 offsets, then nbr, eid and dt bits, little-endian."""
    blk = {"offsets": np.array([5, 6, 8], dtype=np.int64), "nbr": np.array([7, 8, 9], dtype=np.int32),
           "eid": np.array([1, 2, 3], dtype=np.int32), "dt": np.array([1.0, 2.0, 0.5], dtype=np.float32)}
    raw = (np.array([0, 1, 3], dtype="<i8").tobytes() + np.array([7, 8, 9], dtype="<i4").tobytes()
           + np.array([1, 2, 3], dtype="<i4").tobytes() + np.array([1.0, 2.0, 0.5], dtype="<f4").tobytes())
    assert oracle.block_digest(blk) == oracle.fnv1a64(raw)
