"""GPU parity: libtgl.so (sm_100a) against the CPU oracle, bit for bit, through the C ABI.

Every comparison is exact: int32 ids / eids, int64 offsets, float32 dt and ts_edge compared as
bit patterns ("GPU output must match the oracle bit-exactly").  Inputs come from
synth/ (generators only); expected values come only from oracle/.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from synth.tiny import random_graph, random_roots

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tgl():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    import paper_2203_14883_b200 as m
    return m


def cu(a, dtype):
    return torch.as_tensor(np.asarray(a), dtype=dtype).cuda()


def gpu_build(tgl, src, dst, ts, eid, n_nodes, add_rev, with_index=True):
    return tgl.build(cu(src, torch.int32), cu(dst, torch.int32), cu(ts, torch.float32),
                     None if eid is None else cu(eid, torch.int32), n_nodes=n_nodes, add_reverse=add_rev,
                     with_index=with_index)


def assert_tcsr_equal(g, go):
    np.testing.assert_array_equal(g.indptr.cpu().numpy(), go["indptr"])
    np.testing.assert_array_equal(g.nbr.cpu().numpy(), go["nbr"])
    np.testing.assert_array_equal(g.ts.cpu().numpy().view(np.uint32), go["ts"].view(np.uint32))
    np.testing.assert_array_equal(g.eid.cpu().numpy(), go["eid"])


def assert_blocks_equal(blocks, blocks_o, L, what=""):
    assert len(blocks) == len(blocks_o)
    for j, (b, bo) in enumerate(zip(blocks, blocks_o)):
        off, nbr, eid, dt, te = b.trimmed()
        np.testing.assert_array_equal(off.cpu().numpy(), bo["offsets"], err_msg=f"{what} block {j} offsets")
        np.testing.assert_array_equal(nbr.cpu().numpy(), bo["nbr"], err_msg=f"{what} block {j} nbr")
        np.testing.assert_array_equal(eid.cpu().numpy(), bo["eid"], err_msg=f"{what} block {j} eid")
        np.testing.assert_array_equal(dt.cpu().numpy().view(np.uint32), bo["dt"].view(np.uint32),
                                      err_msg=f"{what} block {j} dt")
        if "ts_edge" in bo:
            np.testing.assert_array_equal(te.cpu().numpy().view(np.uint32), bo["ts_edge"].view(np.uint32))


def both(tgl, src, dst, ts, eid, n_nodes, add_rev, roots, rts, fanouts, strategy, S, t_s, seed, base,
         with_index=True):
    go = oracle.build(src, dst, ts, eid, n_nodes=n_nodes, add_reverse=add_rev)
    g = gpu_build(tgl, src, dst, ts, eid, n_nodes, add_rev, with_index)
    assert_tcsr_equal(g, go)
    bo = oracle.sample(go, roots, rts, fanouts=fanouts, strategy=strategy, n_snapshots=S, snapshot_len=t_s,
                       seed=seed, root_key_base=base)
    b = tgl.sample(g, cu(roots, torch.int32), cu(rts, torch.float32), fanouts=fanouts, strategy=strategy,
                   n_snapshots=S, snapshot_len=t_s, seed=seed, root_key_base=base)
    assert_blocks_equal(b, bo, len(fanouts))
    return g, b


# ----------------------------------------------------------------------------- random small graphs
def test_random_graphs_bit_exact(tgl):
    rng = np.random.default_rng(77)
    for case in range(120):
        n_nodes = int(rng.integers(1, 400))
        n_edges = int(rng.integers(0, 5000))
        add_rev = bool(case % 2)
        integer_times = case % 3 != 0
        src, dst, ts, eid = random_graph(case, n_nodes, n_edges, with_eid=bool(case % 5 == 0),
                                         integer_times=integer_times)
        roots, rts = random_roots(case, n_nodes, int(rng.integers(0, 900)), integer_times=integer_times)
        L = 1 + case % 2
        fanouts = [int(rng.integers(1, 12)) for _ in range(L)]
        strategy = int(rng.integers(0, 2))
        S = int(rng.integers(1, 5))
        t_s = math.inf if S == 1 and case % 4 else float(rng.choice([1.0, 2.5, 7.0]))
        seed = int(rng.integers(0, 2**63))
        base = int(rng.integers(0, 2**40))
        both(tgl, src, dst, ts, eid, n_nodes, add_rev, roots, rts, fanouts, strategy, S, t_s, seed, base,
             with_index=case % 7 != 3)


@pytest.mark.parametrize("n_nodes", [1, 2, 255, 256, 257, 65536, 65537, 20_000_000])
def test_build_radix_pass_counts(tgl, n_nodes):
    """1, 2, 3 and 4 LSD passes (8 bits each) and the id-space edges of each."""
    n_edges = 30_000
    rng = np.random.default_rng(n_nodes)
    src = rng.integers(0, n_nodes, n_edges).astype(np.int32)
    dst = rng.integers(0, n_nodes, n_edges).astype(np.int32)
    src[:3] = [0, n_nodes - 1, n_nodes - 1]
    ts = np.sort(rng.integers(0, 100, n_edges)).astype(np.float32)
    for add_rev in (False, True):
        go = oracle.build(src, dst, ts, None, n_nodes=n_nodes, add_reverse=add_rev)
        g = gpu_build(tgl, src, dst, ts, None, n_nodes, add_rev)
        assert_tcsr_equal(g, go)


def test_multi_tile_ragged_and_hub(tgl):
    """Many 256-root tiles with a ragged tail; a hub with 200k edges (deep binary search)."""
    rng = np.random.default_rng(5)
    n_nodes, n_edges = 3000, 400_000
    src = rng.integers(0, n_nodes, n_edges).astype(np.int32)
    src[rng.random(n_edges) < 0.5] = 17                      # hub
    dst = rng.integers(0, n_nodes, n_edges).astype(np.int32)
    ts = np.sort(rng.random(n_edges) * 1e5).astype(np.float32)
    roots = rng.integers(0, n_nodes, 256 * 13 + 37).astype(np.int32)
    roots[::3] = 17
    rts = (rng.random(len(roots)) * 1.1e5).astype(np.float32)
    for strategy in (0, 1):
        for S, t_s in ((1, math.inf), (3, 5000.0)):
            for with_index in (True, False):
                both(tgl, src, dst, ts, None, n_nodes, True, roots, rts, [10, 4], strategy, S, t_s, 3, 1000,
                     with_index=with_index)


def test_wrap_rebuilds_index(tgl):
    """tgl_tcsr_wrap + tgl_tcsr_aux_build over arrays of a built T-CSR give identical samples."""
    src, dst, ts, _ = random_graph(12, 200, 30_000, integer_times=False, t_max=1e4)
    roots, rts = random_roots(12, 200, 3000, integer_times=False, t_max=1e4)
    g = gpu_build(tgl, src, dst, ts, None, 200, True)
    g2 = tgl.wrap(g.indptr.clone(), g.nbr.clone(), g.ts.clone(), g.eid.clone())
    R, T = cu(roots, torch.int32), cu(rts, torch.float32)
    a = tgl.sample(g, R, T, fanouts=[10], n_snapshots=3, snapshot_len=500.0)
    b = tgl.sample(g2, R, T, fanouts=[10], n_snapshots=3, snapshot_len=500.0)
    for x, y in zip(a, b):
        for u, w in zip(x.trimmed()[:4], y.trimmed()[:4]):
            assert torch.equal(u, w)


@pytest.mark.parametrize("k,S,strategy", [(64, 1, 1), (65, 1, 1), (1024, 1, 1), (300, 4, 1), (1, 16, 0),
                                          (7, 16, 1), (1024, 2, 0)])
def test_large_fanouts_and_snapshots(tgl, k, S, strategy):
    """Uniform picks in shared memory (S*k <= 64) and in the global workspace (S*k > 64)."""
    src, dst, ts, _ = random_graph(9, 50, 60_000, integer_times=False, t_max=1000.0)
    roots, rts = random_roots(9, 50, 700, integer_times=False, t_max=1000.0)
    both(tgl, src, dst, ts, None, 50, True, roots, rts, [k], strategy, S, 30.0 if S > 1 else math.inf, 11, 0)


def test_degenerate_inputs(tgl):
    # empty graph, roots present
    both(tgl, [], [], np.zeros(0, np.float32), None, 4, True, [0, 1, 3], np.float32([1, 2, 3]), [5, 5], 1, 1,
         math.inf, 0, 0)
    # no roots
    src, dst, ts, _ = random_graph(1, 10, 100)
    both(tgl, src, dst, ts, None, 10, False, np.zeros(0, np.int32), np.zeros(0, np.float32), [3, 2], 0, 2, 4.0,
         0, 0)
    # single node, self loops only
    both(tgl, [0, 0, 0], [0, 0, 0], np.float32([1, 1, 2]), None, 1, True, [0, 0], np.float32([2, 3]), [2], 0, 1,
         math.inf, 0, 0)


def test_subnormal_dt_is_not_flushed(tgl):
    tiny = np.float32(1.4e-45)
    both(tgl, [0, 0], [1, 2], np.array([0.0, tiny], np.float32), None, 3, False, [0], np.array([2 * tiny], np.float32),
         [5], 0, 1, math.inf, 0, 0)


def test_per_batch_equals_epoch_mode(tgl):
    """Root keys are global root indices (R#7): one call == many per-batch calls, bit for bit."""
    src, dst, ts, _ = random_graph(21, 300, 50_000, integer_times=True, t_max=5000)
    roots, rts = random_roots(21, 300, 6000, integer_times=True, t_max=5000)
    g = gpu_build(tgl, src, dst, ts, None, 300, True)
    R, T = cu(roots, torch.int32), cu(rts, torch.float32)
    for strategy in ("most_recent", "uniform"):
        whole = tgl.sample(g, R, T, fanouts=[10, 10], strategy=strategy, seed=5, root_key_base=0)
        w0 = [x.cpu().numpy() for x in whole[0].trimmed()[1:3]]
        w1 = [x.cpu().numpy() for x in whole[1].trimmed()[1:3]]
        p0, p1 = [[], []], [[], []]
        for a in range(0, 6000, 600):
            part = tgl.sample(g, R[a:a + 600], T[a:a + 600], fanouts=[10, 10], strategy=strategy, seed=5,
                              root_key_base=a)
            for j, x in enumerate(part[0].trimmed()[1:3]):
                p0[j].append(x.cpu().numpy())
            for j, x in enumerate(part[1].trimmed()[1:3]):
                p1[j].append(x.cpu().numpy())
        for j in range(2):
            np.testing.assert_array_equal(np.concatenate(p0[j]), w0[j])
            np.testing.assert_array_equal(np.concatenate(p1[j]), w1[j])
        again = tgl.sample(g, R, T, fanouts=[10, 10], strategy=strategy, seed=5, root_key_base=0)
        np.testing.assert_array_equal(again[1].trimmed()[2].cpu().numpy(), w1[1])   # run-to-run identical


# ----------------------------------------------------------------------------- errors
def test_build_errors(tgl):
    for src, ts, code in (([0, 9], [0.0, 1.0], tgl._lib.ERANGE), ([0, 1], [0.0, float("nan")], tgl._lib.EINVAL),
                          ([0, 1], [-1.0, 1.0], tgl._lib.EINVAL), ([0, 1], [2.0, 1.0], tgl._lib.EUNSORTED)):
        with pytest.raises(tgl.TGLError) as ei:
            gpu_build(tgl, src, [1, 1], np.float32(ts), None, 3, True)
        assert ei.value.code == code


def test_sample_sticky_errors(tgl):
    g = gpu_build(tgl, [0, 1], [1, 0], np.float32([1, 2]), None, 2, True)
    assert tgl.check(g) == 0
    b = tgl.sample(g, cu([0, 5, 1], torch.int32), cu([9, 9, 9], torch.float32), fanouts=[4])
    assert tgl.check(g) == tgl._lib.ERANGE
    assert list(b[0].trimmed()[0].cpu().numpy()) == [0, 2, 2, 4]
    assert tgl.check(g) == 0                                          # cleared
    tgl.sample(g, cu([0], torch.int32), cu([float("nan")], torch.float32), fanouts=[4])
    assert tgl.check(g) == tgl._lib.EINVAL


# ----------------------------------------------------------------------------- gather
@pytest.mark.parametrize("cols,dtype", [(1, np.float32), (3, np.float32), (100, np.float32), (428, np.float32),
                                        (3, np.uint8), (5, np.int16), (2, np.float64)])
def test_gather_bit_exact(tgl, cols, dtype):
    rng = np.random.default_rng(cols)
    rows = 3000
    table = (rng.standard_normal((rows, cols)) * 100).astype(dtype)
    ids = rng.integers(-1, rows, 10_001).astype(np.int32)
    want, err = oracle.gather(ids, table)
    assert err == 0
    got = tgl.gather(cu(ids, torch.int32), [torch.from_numpy(table).cuda()])[0]
    np.testing.assert_array_equal(got.cpu().numpy().view(np.uint8), want.view(np.uint8))
    assert tgl.check(None) == 0


def test_gather_device_count_and_range_error(tgl):
    table = torch.arange(40, dtype=torch.float32, device="cuda").reshape(10, 4)
    ids = cu([1, 2, 3, 99, 5], torch.int32)
    n_dev = torch.tensor([3], dtype=torch.int64, device="cuda")
    out = torch.full((5, 4), -7.0, device="cuda")
    tgl.gather(ids, [table], n_ids_dev=n_dev, outs=[out])
    assert tgl.check(None) == 0
    np.testing.assert_array_equal(out[:3].cpu().numpy(), table[1:4].cpu().numpy())
    assert (out[3:] == -7.0).all()                                    # beyond *n_ids_dev untouched
    tgl.gather(ids, [table])
    assert tgl.check(None) == tgl._lib.ERANGE


# ----------------------------------------------------------------------------- shard bucketing
def test_shard_bucket_stable(tgl):
    rng = np.random.default_rng(3)
    V, world = 100_000, 8
    roots = rng.integers(0, V, 50_000).astype(np.int32)
    splits = np.sort(rng.choice(np.arange(1, V), world - 1, replace=False))
    splits = np.concatenate([[0], splits, [V]]).astype(np.int64)
    perm, counts = tgl.shard_bucket(cu(roots, torch.int32), cu(splits, torch.int64), world)
    owner = np.searchsorted(splits, roots, side="right") - 1
    want = np.argsort(owner, kind="stable")
    np.testing.assert_array_equal(perm.cpu().numpy(), want)
    np.testing.assert_array_equal(counts.cpu().numpy(), np.bincount(owner, minlength=world))


# ----------------------------------------------------------------------------- golden fixtures
@pytest.mark.parametrize("name", ["fig3.json", "ties.json", "r3_hops.json"])
def test_golden_examples_on_gpu(tgl, golden_dir, name):
    """The paper's worked examples (Fig. 3), the tie rule (R#8) and the R#3 hop-window
    example, through the C ABI: expected values are the fixtures' hand-worked ones, not the oracle's."""
    import json
    import os
    gd = json.load(open(os.path.join(golden_dir, name)))
    e = gd["edges"]
    g = gpu_build(tgl, e["src"], e["dst"], np.float32(e["ts"]), None, gd["n_nodes"], bool(gd["add_reverse"]))
    for case in gd["cases"]:
        t_s = math.inf if case["snapshot_len"] == "inf" else float(case["snapshot_len"])
        blocks = tgl.sample(g, cu([case["root"]], torch.int32), cu([case["t"]], torch.float32),
                            fanouts=case["fanouts"], strategy=case["strategy"], n_snapshots=case["n_snapshots"],
                            snapshot_len=t_s, seed=0, root_key_base=0)
        assert len(blocks) == len(case["blocks"]), case["what"]
        for b, want in zip(blocks, case["blocks"]):
            off, nbr, eid, dt, _ = b.trimmed()
            assert nbr.cpu().tolist() == want["nbr"], case["what"]
            assert eid.cpu().tolist() == want["eid"], case["what"]
            assert [float(x) for x in dt.cpu().tolist()] == want["dt"], case["what"]
            assert off.cpu().tolist() == [0, len(want["nbr"])], case["what"]


@pytest.mark.parametrize("strategy", ["most_recent", "uniform"])
def test_forked_snapshot_chains_equal_captured_sequential(tgl, strategy):
    """S > 1, L > 1: eager calls fork the layer >= 1 snapshot chains onto side streams; under CUDA-graph
    capture they run in order on the caller's stream.  Both orders give the oracle's blocks, bit for bit,
    on a non-default caller stream."""
    src, dst, ts, _ = random_graph(31, 200, 40_000, integer_times=True, t_max=4000)
    roots, rts = random_roots(31, 200, 3000, integer_times=True, t_max=4000)
    g = gpu_build(tgl, src, dst, ts, None, 200, True)
    go = oracle.build(src, dst, ts, None, n_nodes=200, add_reverse=True)
    bo = oracle.sample(go, roots, rts, fanouts=[6, 4], strategy=0 if strategy == "most_recent" else 1, n_snapshots=3,
                       snapshot_len=300.0, seed=9, root_key_base=0)
    R, T = cu(roots, torch.int32), cu(rts, torch.float32)
    smp = tgl.Sampler(g, 3000, [6, 4], strategy, 3, 300.0)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        eager = [[x.clone() for x in b.trimmed()[:4]] for b in smp.run(R, T, seed=9, root_key_base=0)]
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            blocks = smp.run(R, T, seed=9, root_key_base=0)
    for b in blocks:  # poison the outputs, then replay the captured (sequential) calls
        b.nbr.fill_(-7)
    graph.replay()
    torch.cuda.synchronize()
    for j, (e, b, o) in enumerate(zip(eager, blocks, bo)):
        c = b.trimmed()[:4]
        for u, w in zip(e, c):
            assert torch.equal(u, w), f"block {j}"
        np.testing.assert_array_equal(e[1].cpu().numpy(), o["nbr"], err_msg=f"block {j}")
        np.testing.assert_array_equal(e[3].cpu().numpy().view(np.uint32), o["dt"].view(np.uint32))
