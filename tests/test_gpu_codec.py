"""GPU parity of the T-CSR time codec (tsindex.cuh "time codes") against the
CPU oracle, bit for bit, through the C ABI.

The codec is a lossless re-encoding of the aux buffer (7-bit time codes, 54 fence codes per node
record, 8-byte packed slot records) used when a graph has at most 127 distinct timestamps -- MAG's
publication years (Table 3 max(t) = 120).  Sampled blocks must not change: every
case here is compared with the oracle, and the codec's on/off decision is checked at its
boundaries (127 vs 128 distinct times, -0.0, one distinct time) and for both record forms
(packed, and 12-byte records when the widths exceed 64 bits).  Expected values come only from
oracle/; inputs from synth/."""
import math

import numpy as np
import pytest
import torch

import oracle
from synth.tiny import random_roots

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tgl():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    import paper_2203_14883_b200 as m
    return m


def cu(a, dtype):
    return torch.as_tensor(np.asarray(a), dtype=dtype).cuda()


def _blocks_equal(b, bo, what):
    assert len(b) == len(bo)
    for j, (x, y) in enumerate(zip(b, bo)):
        off, nbr, eid, dt, te = x.trimmed()
        np.testing.assert_array_equal(off.cpu().numpy(), y["offsets"], err_msg=f"{what} block {j} offsets")
        np.testing.assert_array_equal(nbr.cpu().numpy(), y["nbr"], err_msg=f"{what} block {j} nbr")
        np.testing.assert_array_equal(eid.cpu().numpy(), y["eid"], err_msg=f"{what} block {j} eid")
        np.testing.assert_array_equal(dt.cpu().numpy().view(np.uint32), y["dt"].view(np.uint32),
                                      err_msg=f"{what} block {j} dt")
        if "ts_edge" in y and te is not None:
            np.testing.assert_array_equal(te.cpu().numpy().view(np.uint32), y["ts_edge"].view(np.uint32),
                                          err_msg=f"{what} block {j} ts_edge")


def _stream(seed, n_nodes, n_edges, values, hub_frac=0.3):
    """chronological stream whose times are drawn from `values` (sorted), with hubs"""
    rng = np.random.default_rng(seed)
    hubs = rng.integers(0, n_nodes, size=max(1, n_nodes // 16))
    pick = rng.random(n_edges) < hub_frac
    src = np.where(pick, rng.choice(hubs, size=n_edges), rng.integers(0, n_nodes, size=n_edges)).astype(np.int32)
    dst = rng.integers(0, n_nodes, size=n_edges).astype(np.int32)
    ts = np.sort(rng.choice(np.asarray(values, dtype=np.float32), size=n_edges)).astype(np.float32)
    return src, dst, ts


def _check(tgl, src, dst, ts, eid, n_nodes, add_rev, roots, rts, *, expect_codes, expect_packed=None,
           cases=(([10], 0, 3, 5.0), ([10], 0, 1, math.inf), ([4, 3], 1, 1, math.inf), ([5, 3], 0, 2, 7.0),
                  ([6], 1, 3, 2.5))):
    go = oracle.build(src, dst, ts, eid, n_nodes=n_nodes, add_reverse=add_rev)
    g = tgl.build(cu(src, torch.int32), cu(dst, torch.int32), cu(ts, torch.float32),
                  None if eid is None else cu(eid, torch.int32), n_nodes=n_nodes, add_reverse=add_rev)
    c = g.codec
    assert c["n_codes"] == expect_codes, c
    if expect_packed is not None:
        assert c["packed"] == expect_packed, c
    for fan, strat, S, t_s in cases:
        bo = oracle.sample(go, roots, rts, fanouts=fan, strategy=strat, n_snapshots=S, snapshot_len=t_s, seed=11,
                           root_key_base=5)
        b = tgl.sample(g, cu(roots, torch.int32), cu(rts, torch.float32), fanouts=fan, strategy=strat,
                       n_snapshots=S, snapshot_len=t_s, seed=11, root_key_base=5)
        _blocks_equal(b, bo, f"D={expect_codes} fan={fan} strat={strat} S={S}")
    assert tgl.check(g) == 0
    return g


@pytest.mark.parametrize("D", [1, 2, 17, 121, 127])
def test_codec_on_bit_exact(tgl, D):
    """<= 127 distinct times: codec on, packed records (small ids), blocks equal the oracle's."""
    values = np.arange(D, dtype=np.float32) * 1.0
    src, dst, ts = _stream(D, 3000, 40_000, values)
    roots, rts = random_roots(D, 3000, 9000, t_max=float(D))
    _check(tgl, src, dst, ts, None, 3000, True, roots, rts, expect_codes=D, expect_packed=True)


def test_codec_fractional_times(tgl):
    """non-integer times (few distinct values) code the same way: the dictionary holds the floats"""
    values = np.float32(0.1) * np.arange(120, dtype=np.float32) + np.float32(1e-3)
    src, dst, ts = _stream(5, 2000, 30_000, values)
    rng = np.random.default_rng(6)
    roots = rng.integers(0, 2000, 7000).astype(np.int32)
    rts = rng.choice(np.concatenate([values, values + np.float32(0.05)]), 7000).astype(np.float32)
    _check(tgl, src, dst, ts, None, 2000, True, roots, rts, expect_codes=int(len(np.unique(ts))),
           cases=(([10], 0, 3, 0.3), ([10], 0, 2, 0.1), ([3, 3], 1, 1, math.inf)))


def test_codec_off_at_128_and_minus_zero(tgl):
    """128 distinct times: no time codes, but integer times pack (packed = 2); a -0.0 time: neither;
    same blocks"""
    values = np.arange(128, dtype=np.float32)
    src, dst, ts = _stream(7, 1500, 20_000, values)
    ts[:128] = values  # every value present
    ts = np.sort(ts)
    roots, rts = random_roots(7, 1500, 4000, t_max=128.0)
    g = _check(tgl, src, dst, ts, None, 1500, True, roots, rts, expect_codes=0, expect_packed=2)
    src, dst, ts = _stream(8, 800, 5000, np.arange(10, dtype=np.float32))
    ts[: np.sum(ts == 0)] = np.float32(-0.0)  # the zeros become -0.0 (still chronological)
    roots, rts = random_roots(8, 800, 2000, t_max=10.0)
    _check(tgl, src, dst, ts, None, 800, True, roots, rts, expect_codes=0, expect_packed=0)


def test_codec_fence_boundaries(tgl):
    """node degrees around the 54 fence codes (53, 54, 55, 106, 107, 108, 2000, 20000: a gap longer
    than the 16-ary index threshold) and cut times at, between and beyond the node's times"""
    degs = [0, 1, 2, 5, 53, 54, 55, 106, 107, 108, 2000, 20_000]
    src, dst, ts = [], [], []
    rng = np.random.default_rng(3)
    for v, d in enumerate(degs):
        src.append(np.full(d, v, np.int32))
        dst.append(rng.integers(0, len(degs), d).astype(np.int32))
        ts.append(rng.integers(0, 100, d).astype(np.float32))
    src, dst, ts = np.concatenate(src), np.concatenate(dst), np.concatenate(ts)
    order = np.argsort(ts, kind="stable")
    src, dst, ts = src[order], dst[order], ts[order]
    n = len(degs)
    roots = np.repeat(np.arange(n, dtype=np.int32), 110)
    rts = np.tile(np.arange(-2, 108, dtype=np.float32), n)
    _check(tgl, src, dst, ts, None, n, False, roots, rts, expect_codes=int(len(np.unique(ts))),
           cases=(([10], 0, 3, 5.0), ([10], 0, 4, 1.0), ([64], 0, 2, 20.0), ([10], 1, 3, 5.0), ([7, 2], 0, 3, 3.0)))


def test_codec_wide_ids_unpacked(tgl):
    """ids too wide for an 8-byte record (31-bit neighbour ids + 32-bit eid spans, via
    tgl_tcsr_wrap / tgl_tcsr_aux_build over given arrays): codec on with 12-byte records"""
    src, dst, ts = _stream(9, 1000, 20_000, np.arange(30, dtype=np.float32))
    rng = np.random.default_rng(10)
    eid = rng.integers(-2**31, 2**31 - 1, size=len(src), dtype=np.int64).astype(np.int32)
    go = oracle.build(src, dst, ts, eid, n_nodes=1000, add_reverse=True)
    wide = oracle.TCSR(indptr=go["indptr"], nbr=(go["nbr"].astype(np.int64) + 2**30 + 12345).astype(np.int32),
                       ts=go["ts"], eid=go["eid"])
    g = tgl.wrap(cu(wide["indptr"], torch.int64), cu(wide["nbr"], torch.int32), cu(wide["ts"], torch.float32),
                 cu(wide["eid"], torch.int32))
    assert g.codec == {"n_codes": 30, "packed": False}
    roots, rts = random_roots(9, 1000, 5000, t_max=30.0)
    for fan, strat, S, t_s in (([10], 0, 3, 4.0), ([10], 1, 1, math.inf)):
        bo = oracle.sample(wide, roots, rts, fanouts=fan, strategy=strat, n_snapshots=S, snapshot_len=t_s, seed=2)
        b = tgl.sample(g, cu(roots, torch.int32), cu(rts, torch.float32), fanouts=fan, strategy=strat,
                       n_snapshots=S, snapshot_len=t_s, seed=2)
        _blocks_equal(b, bo, f"wide {fan} {strat}")
    # the same arrays with narrow ids: packed
    g2 = tgl.wrap(cu(go["indptr"], torch.int64), cu(go["nbr"], torch.int32), cu(go["ts"], torch.float32),
                  cu((go["eid"].astype(np.int64) & 0xFFFFF).astype(np.int32), torch.int32))
    assert g2.codec == {"n_codes": 30, "packed": True}


def test_codec_fused_gather_and_variants(tgl):
    """packed records through the fused gather (copy kernel OUTX 2), the validity path (codec
    structures bypassed) and root-time hops / replacement / dedup variants"""
    src, dst, ts = _stream(12, 2500, 30_000, np.arange(121, dtype=np.float32))
    go = oracle.build(src, dst, ts, n_nodes=2500, add_reverse=True)
    g = tgl.build(cu(src, torch.int32), cu(dst, torch.int32), cu(ts, torch.float32), n_nodes=2500, add_reverse=True)
    assert g.codec == {"n_codes": 121, "packed": True}
    roots, rts = random_roots(12, 2500, 6000, t_max=121.0)
    r, t = cu(roots, torch.int32), cu(rts, torch.float32)
    node_tab = torch.arange(2500 * 8, dtype=torch.float32, device="cuda").reshape(2500, 8)
    edge_tab = torch.arange(30_000 * 3, dtype=torch.float32, device="cuda").reshape(30_000, 3)
    spec = [(node_tab, "node"), (edge_tab, "edge")]
    for fan, strat in (([10], "most_recent"), ([4, 5], "uniform")):
        smp = tgl.Sampler(g, r.numel(), fan, strat, fused_gather=spec)
        blocks = smp.run(r, t, seed=3, root_key_base=0)
        bo = oracle.sample(go, roots, rts, fanouts=fan, strategy=0 if strat == "most_recent" else 1, seed=3)
        _blocks_equal(blocks, bo, f"fused {strat}")
        last = blocks[-1]
        n = int(last.nnz_dev.item())
        for (tab, by), got in zip(spec, smp.fused_outs):
            want = tgl.gather(last.nbr if by == "node" else last.eid, [tab], n_ids_dev=last.nnz_dev)[0]
            assert torch.equal(got[:n], want[:n])
    valid = np.random.default_rng(13).integers(0, 2**32, size=(30_000 + 31) // 32, dtype=np.uint64).astype(np.uint32)
    for kw in (dict(edge_valid=valid), dict(hop_time="root"), dict(replacement=True), dict(dedup=True)):
        fan, strat = ([6, 3], 1)
        bo = oracle.sample(go, roots, rts, fanouts=fan, strategy=strat, seed=4, **kw)
        kw_g = dict(kw)
        if "edge_valid" in kw_g:
            kw_g["edge_valid"] = cu(valid.view(np.int32), torch.int32)
        b = tgl.sample(g, r, t, fanouts=fan, strategy="uniform", seed=4, **kw_g)
        _blocks_equal(b, bo, f"variant {list(kw)}")
    assert tgl.check(g) == 0


def test_codec_sticky_errors(tgl):
    """out-of-range roots read as empty lists (count 0 + sticky ERANGE) and NaN root times as EINVAL
    on a codec graph, as without the codec"""
    src, dst, ts = _stream(14, 50, 2000, np.arange(20, dtype=np.float32))
    g = tgl.build(cu(src, torch.int32), cu(dst, torch.int32), cu(ts, torch.float32), n_nodes=50, add_reverse=True)
    assert g.codec["n_codes"] == 20
    go = oracle.build(src, dst, ts, n_nodes=50, add_reverse=True)
    roots = np.array([3, 50, 7, -1, 9] * 60, np.int32)
    rts = np.array([15, 15, 19, 4, 12] * 60, np.float32)
    b = tgl.sample(g, cu(roots, torch.int32), cu(rts, torch.float32), fanouts=[5], n_snapshots=3, snapshot_len=2.0)
    assert tgl.check(g) == tgl._lib.ERANGE
    ok = (roots >= 0) & (roots < 50)
    bo = oracle.sample(go, np.where(ok, roots, 0), np.where(ok, rts, -1.0).astype(np.float32), fanouts=[5],
                       strategy=0, n_snapshots=3, snapshot_len=2.0)
    _blocks_equal(b, bo, "out-of-range roots")  # a root at time -1 selects nothing, like a bad id
    tgl.sample(g, cu([0], torch.int32), cu([float("nan")], torch.float32), fanouts=[4])
    assert tgl.check(g) == tgl._lib.EINVAL


def test_codec_empty_and_foreign_aux(tgl):
    """an empty stream builds (no codec) and samples nothing; tgl_tcsr_wrap rejects an aux buffer
    that no aux build filled (EINVAL), instead of reading garbage codec widths"""
    import ctypes
    from paper_2203_14883_b200 import _lib
    e = np.zeros(0, np.int32)
    g = tgl.build(cu(e, torch.int32), cu(e, torch.int32), cu(np.zeros(0, np.float32), torch.float32), n_nodes=5,
                  add_reverse=True)
    assert g.codec == {"n_codes": 0, "packed": 0}
    b = tgl.sample(g, cu([0, 4], torch.int32), cu([3.0, 7.0], torch.float32), fanouts=[4], n_snapshots=2,
                   snapshot_len=1.0)
    for x in b:
        off, nbr, _, _, _ = x.trimmed()
        assert off.cpu().tolist() == [0, 0, 0] and nbr.numel() == 0
    src, dst, ts = _stream(15, 100, 1000, np.arange(5, dtype=np.float32))
    g2 = tgl.build(cu(src, torch.int32), cu(dst, torch.int32), cu(ts, torch.float32), n_nodes=100, add_reverse=True)
    junk = torch.full((g2.index.numel(),), 0x5A, dtype=torch.uint8, device="cuda")
    h = ctypes.c_void_p()
    rc = tgl._L.tgl_tcsr_wrap(g2.indptr.data_ptr(), g2.nbr.data_ptr(), g2.ts.data_ptr(), g2.eid.data_ptr(),
                              junk.data_ptr(), junk.numel(), 100, g2.n_stored, ctypes.byref(h))
    assert rc == _lib.EINVAL


def test_integer_time_packing(tgl):
    """GDELT-like integer ticks (more than 127 distinct): 8-byte records with integer times
    (packed = 2) -- uniform 2-layer and most_recent S = 3 equal the oracle; real-valued times or a
    time >= 2^24 do not pack"""
    rng = np.random.default_rng(21)
    for vmax, expect in ((180_000, 2), (2**24 + 50, 0)):
        src = rng.integers(0, 700, 30_000).astype(np.int32)
        dst = rng.integers(0, 700, 30_000).astype(np.int32)
        ts = np.sort(rng.integers(0, vmax, 30_000)).astype(np.float32)
        ts[-1] = np.float32(vmax)  # the largest time present (2^24 + 50 -> 2^24 + 50 rounds to an even float)
        roots, rts = src[::7].copy(), (ts[::7] + 1).astype(np.float32)
        _check(tgl, src, dst, ts, None, 700, False, roots, rts, expect_codes=0, expect_packed=expect,
               cases=(([10, 10], 1, 1, math.inf), ([10], 0, 3, 5000.0), ([4, 3], 0, 1, math.inf)))
    src, dst, ts = _stream(22, 500, 8000, np.float32(0.5) + np.arange(300, dtype=np.float32))
    roots, rts = random_roots(22, 500, 3000, t_max=300.0)
    _check(tgl, src, dst, ts, None, 500, True, roots, rts, expect_codes=0, expect_packed=0)
