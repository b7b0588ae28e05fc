"""GPU parity of the sampler variants (tgl_sample_ex, R#23, R#24)
against the CPU oracle, bit for bit, on random graphs (multi-tile, ragged, hubs, 1-3 layers,
1-4 snapshots), plus the option validation of the C ABI."""
import ctypes
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


@pytest.mark.parametrize("hop_time,replacement", [("root", False), ("edge", True), ("root", True)])
def test_variants_bit_exact(tgl, hop_time, replacement):
    rng = np.random.default_rng(31 + replacement + 2 * (hop_time == "root"))
    for case in range(60):
        n_nodes = int(rng.integers(1, 500))
        n_edges = int(rng.integers(0, 6000))
        add_rev = bool(case % 2)
        src, dst, ts, eid = random_graph(900 + case, n_nodes, n_edges, integer_times=case % 3 != 0)
        roots, rts = random_roots(900 + case, n_nodes, int(rng.integers(0, 1500)), integer_times=case % 3 != 0)
        L = 1 + case % 3
        fanouts = [int(rng.integers(1, 12)) for _ in range(L)]
        strategy = 1 if replacement else int(rng.integers(0, 2))
        S = int(rng.integers(1, 5))
        t_s = math.inf if S == 1 and case % 4 else float(rng.choice([1.0, 2.5, 7.0]))
        seed, base = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**40))
        go = oracle.build(src, dst, ts, eid, n_nodes=n_nodes, add_reverse=add_rev)
        g = tgl.build(cu(src, torch.int32), cu(dst, torch.int32), cu(ts, torch.float32), None,
                      n_nodes=n_nodes, add_reverse=add_rev, with_index=case % 5 != 2)
        bo = oracle.sample(go, roots, rts, fanouts=fanouts, strategy=strategy, n_snapshots=S, snapshot_len=t_s,
                           seed=seed, root_key_base=base, hop_time=hop_time, replacement=replacement)
        try:
            b = tgl.sample(g, cu(roots, torch.int32), cu(rts, torch.float32), fanouts=fanouts, strategy=strategy,
                           n_snapshots=S, snapshot_len=t_s, seed=seed, root_key_base=base, hop_time=hop_time,
                           replacement=replacement)
        except Exception as ex:
            raise AssertionError(f"case {case}: L={L} fanouts={fanouts} strategy={strategy} S={S} t_s={t_s} "
                                 f"roots={len(roots)}") from ex
        for j, (x, o) in enumerate(zip(b, bo)):
            off, nbr, e, dt, _ = x.trimmed()
            np.testing.assert_array_equal(off.cpu().numpy(), o["offsets"], err_msg=f"case {case} block {j}")
            np.testing.assert_array_equal(nbr.cpu().numpy(), o["nbr"])
            np.testing.assert_array_equal(e.cpu().numpy(), o["eid"])
            np.testing.assert_array_equal(dt.cpu().numpy().view(np.uint32), o["dt"].view(np.uint32))


def test_keyed_variant_equals_base_keys(tgl):
    """tgl_sample_ex with explicit keys root_key_base + i == with root_key_base (R#7)."""
    src, dst, ts, _ = random_graph(5, 300, 5000)
    roots, rts = random_roots(5, 300, 700)
    g = tgl.build(cu(src, torch.int32), cu(dst, torch.int32), cu(ts, torch.float32), None, n_nodes=300,
                  add_reverse=True)
    smp = tgl.Sampler(g, 700, [5, 3], "uniform", hop_time="root", replacement=True)
    a = [x.trimmed() for x in smp.run(cu(roots, torch.int32), cu(rts, torch.float32), seed=9, root_key_base=1000)]
    a = [[t.cpu().numpy() for t in x[:4]] for x in a]
    keys = torch.arange(1000, 1700, dtype=torch.int64, device="cuda")
    b = [x.trimmed() for x in smp.run(cu(roots, torch.int32), cu(rts, torch.float32), seed=9, root_keys=keys)]
    for x, y in zip(a, b):
        for u, v in zip(x, y[:4]):
            np.testing.assert_array_equal(u, v.cpu().numpy())


def test_option_validation(tgl):
    from paper_2203_14883_b200 import _lib
    L_ = _lib.load()
    src, dst, ts, _ = random_graph(1, 10, 50)
    g = tgl.build(cu(src, torch.int32), cu(dst, torch.int32), cu(ts, torch.float32), None, n_nodes=10,
                  add_reverse=False)
    smp = tgl.Sampler(g, 4, [3], "most_recent")
    r, t = cu([1, 2, 3, 4], torch.int32), cu([10.0, 20.0, 30.0, 40.0], torch.float32)
    fan = (ctypes.c_int32 * 1)(3)

    def call(opts, strategy=0):
        return L_.tgl_sample_ex(g.handle, r.data_ptr(), t.data_ptr(), None, 4, 1, fan, strategy, 1, math.inf, 0, 0,
                                ctypes.byref(opts), smp._c_blocks, None, smp.workspace.data_ptr(), smp.ws_bytes, None)
    assert call(_lib.SampleOptions(0, 0)) == 0
    assert call(_lib.SampleOptions(2, 0)) == -1            # unknown hop_time
    assert call(_lib.SampleOptions(0, 1)) == -1            # replacement with most_recent
    o = _lib.SampleOptions(0, 0)
    o.reserved[3] = 1
    assert call(o) == -1                                   # reserved words must be zero
    assert call(_lib.SampleOptions(0, 0, 1)) == -1         # dedup without dedup blocks
    torch.cuda.synchronize()


@pytest.mark.parametrize("hop_time", ["edge", "root"])
def test_dedup_bit_exact(tgl, hop_time):
    """R#27: distinct (node, hop time) lists, src_index and the deduplicated next layers vs oracle."""
    rng = np.random.default_rng(55 + (hop_time == "root"))
    for case in range(40):
        n_nodes = int(rng.integers(1, 400))
        src, dst, ts, _ = random_graph(1300 + case, n_nodes, int(rng.integers(0, 6000)), integer_times=True,
                                       t_max=float(rng.choice([6.0, 50.0])))
        roots, rts = random_roots(1300 + case, n_nodes, int(rng.integers(0, 1500)), integer_times=True, t_max=50.0)
        L = 1 + case % 3
        fanouts = [int(rng.integers(1, 12)) for _ in range(L)]
        strategy = int(rng.integers(0, 2))
        S = 1 if L > 1 else int(rng.integers(1, 4))
        t_s = math.inf if S == 1 else 7.0
        seed, base = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**40))
        add_rev = bool(case % 2)
        go = oracle.build(src, dst, ts, None, n_nodes=n_nodes, add_reverse=add_rev)
        g = tgl.build(cu(src, torch.int32), cu(dst, torch.int32), cu(ts, torch.float32), None, n_nodes=n_nodes,
                      add_reverse=add_rev)
        bo = oracle.sample(go, roots, rts, fanouts=fanouts, strategy=strategy, n_snapshots=S, snapshot_len=t_s,
                           seed=seed, root_key_base=base, hop_time=hop_time, dedup=True)
        b = tgl.sample(g, cu(roots, torch.int32), cu(rts, torch.float32), fanouts=fanouts, strategy=strategy,
                       n_snapshots=S, snapshot_len=t_s, seed=seed, root_key_base=base, hop_time=hop_time, dedup=True)
        for j, (x, o) in enumerate(zip(b, bo)):
            off, nbr, e, dt, _ = x.trimmed()
            np.testing.assert_array_equal(off.cpu().numpy(), o["offsets"], err_msg=f"case {case} block {j}")
            np.testing.assert_array_equal(nbr.cpu().numpy(), o["nbr"])
            np.testing.assert_array_equal(e.cpu().numpy(), o["eid"])
            np.testing.assert_array_equal(dt.cpu().numpy().view(np.uint32), o["dt"].view(np.uint32))
            nnz, nu = len(o["nbr"]), int(x.n_uniq_dev.item())
            assert nu == len(o["uniq_node"])
            np.testing.assert_array_equal(x.src_index[:nnz].cpu().numpy(), o["src_index"])
            np.testing.assert_array_equal(x.uniq_node[:nu].cpu().numpy(), o["uniq_node"])
            np.testing.assert_array_equal(x.uniq_ts[:nu].cpu().numpy().view(np.uint32), o["uniq_ts"].view(np.uint32))


def _np_mask(rng, n, frac):
    bits = rng.random(max(n, 1)) < frac
    words = np.zeros((len(bits) + 31) // 32, dtype=np.uint32)
    idx = np.nonzero(bits)[0]
    np.bitwise_or.at(words, idx >> 5, (np.uint32(1) << (idx & 31).astype(np.uint32)))
    return words


@pytest.mark.parametrize("strategy,replacement", [(0, False), (1, False), (1, True)])
def test_edge_validity_bit_exact(tgl, strategy, replacement):
    """R#28: invalid edges are not candidates -- GPU vs oracle on random graphs and masks."""
    rng = np.random.default_rng(90 + strategy + 2 * replacement)
    for case in range(40):
        n_nodes = int(rng.integers(1, 400))
        n_edges = int(rng.integers(0, 6000))
        src, dst, ts, eid = random_graph(1500 + case, n_nodes, n_edges, integer_times=case % 3 != 0)
        roots, rts = random_roots(1500 + case, n_nodes, int(rng.integers(0, 1500)), integer_times=case % 3 != 0)
        L = 1 + case % 3
        fanouts = [int(rng.integers(1, 12)) for _ in range(L)]
        S = int(rng.integers(1, 5))
        t_s = math.inf if S == 1 and case % 4 else float(rng.choice([1.0, 2.5, 7.0]))
        seed, base = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**40))
        add_rev = bool(case % 2)
        mask = _np_mask(rng, n_edges, float(rng.choice([0.0, 0.25, 0.7, 1.0])))
        go = oracle.build(src, dst, ts, None, n_nodes=n_nodes, add_reverse=add_rev)
        g = tgl.build(cu(src, torch.int32), cu(dst, torch.int32), cu(ts, torch.float32), None, n_nodes=n_nodes,
                      add_reverse=add_rev)
        bo = oracle.sample(go, roots, rts, fanouts=fanouts, strategy=strategy, n_snapshots=S, snapshot_len=t_s,
                           seed=seed, root_key_base=base, replacement=replacement, edge_valid=mask)
        b = tgl.sample(g, cu(roots, torch.int32), cu(rts, torch.float32), fanouts=fanouts, strategy=strategy,
                       n_snapshots=S, snapshot_len=t_s, seed=seed, root_key_base=base, replacement=replacement,
                       edge_valid=torch.from_numpy(mask.view(np.int32)).cuda())
        for j, (x, o) in enumerate(zip(b, bo)):
            off, nbr, e, dt, _ = x.trimmed()
            np.testing.assert_array_equal(off.cpu().numpy(), o["offsets"], err_msg=f"case {case} block {j}")
            np.testing.assert_array_equal(nbr.cpu().numpy(), o["nbr"])
            np.testing.assert_array_equal(e.cpu().numpy(), o["eid"])
            np.testing.assert_array_equal(dt.cpu().numpy().view(np.uint32), o["dt"].view(np.uint32))


def test_edge_valid_set(tgl):
    rng = np.random.default_rng(3)
    n_bits = 5000
    mask = _np_mask(rng, n_bits, 0.5)
    g_mask = torch.from_numpy(mask.view(np.int32).copy()).cuda()
    ids = rng.integers(-5, n_bits + 5, 800).astype(np.int32)
    tgl.edge_valid_set(g_mask, torch.from_numpy(ids).cuda(), False, n_bits=n_bits)
    ok = ids[(ids >= 0) & (ids < n_bits)]
    np.bitwise_and.at(mask, ok >> 5, ~(np.uint32(1) << (ok & 31).astype(np.uint32)))
    np.testing.assert_array_equal(g_mask.cpu().numpy().view(np.uint32), mask)
    tgl.edge_valid_set(g_mask, torch.from_numpy(ids).cuda(), True, n_bits=n_bits)
    np.bitwise_or.at(mask, ok >> 5, (np.uint32(1) << (ok & 31).astype(np.uint32)))
    np.testing.assert_array_equal(g_mask.cpu().numpy().view(np.uint32), mask)
