"""GPU parity of the TIMED launch configuration: one tgl_sample call spanning thousands of 256-root
tiles (so the copy kernel's tile bases go through the hyper totals: >= 4,096 tiles per chain), as
bench.py times it, compared element by element with the oracle run per batch (key base = the
batch's global root index, R#7) and per batch through tgl_block_digest against the oracle's
FNV-1a digests.  Expected values come only from oracle/."""
import numpy as np
import pytest
import torch

import bench
from synth import configs as C

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tgl():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_2203_14883_b200 as m
    return m


def _check_call(tgl, cfg, g, go, r, t, key0):
    B = cfg.batch
    L, S = len(cfg.fanouts), cfg.n_snapshots
    smp = tgl.Sampler(g, r.numel(), cfg.fanouts, cfg.strategy, S, cfg.snapshot_len)
    blocks = smp.run(r, t, seed=cfg.sampler_seed, root_key_base=key0)
    assert tgl.check(g) == 0
    per_batch, _ = bench.oracle_batches(go, cfg, r.cpu().numpy(), t.cpu().numpy(), key0, n_threads=16)
    ok, msg = bench.compare_blocks(blocks, bench.concat_batches(per_batch, L * S))
    assert ok, msg
    gd = bench.gpu_batch_digests(tgl, blocks, r.numel(), B, L, S)
    od = bench.oracle_batch_digests(per_batch, L * S)
    np.testing.assert_array_equal(gd, od)
    return blocks


def test_c2_whole_epoch_one_call(tgl):
    """C2 (2-layer uniform 10/10): the whole epoch, 2.02 M roots = 7,881 layer-0 tiles and ~78,000
    layer-1 tiles, in ONE call."""
    cfg = C.CONFIGS["C2"]
    src, dst, ts = C.edges("C2", cfg, device="cuda")
    g = tgl.build(src, dst, ts, n_nodes=cfg.n_nodes, add_reverse=cfg.add_reverse)
    go, _ = bench.oracle_graph(cfg, src, dst, ts, [])
    n = cfg.n_roots_epoch // cfg.batch * cfg.batch
    assert (n + 255) // 256 > 4096
    r, t = C.roots(cfg, src, dst, ts, 0, n)
    _check_call(tgl, cfg, g, go, r, t, 0)


def test_c5_bench_call(tgl):
    """C5: the exact bench step -- 2,048 batches x 4,000 roots = 8,192,000 roots = 32,000 tiles in
    one call -- at two positions of the epoch (middle, end: long histories)."""
    cfg = C.CONFIGS["C5"]
    src, dst, ts = C.edges("C5", cfg, device="cuda")
    g = tgl.build(src, dst, ts, n_nodes=cfg.n_nodes, add_reverse=True)
    chunk = 2048 * cfg.batch
    starts = bench.chunk_starts(cfg.n_roots_epoch, chunk, 3, cfg.batch)[1:]
    rts = [C.roots(cfg, src, dst, ts, s0, chunk) for s0 in starts]
    go, _ = bench.oracle_graph(cfg, src, dst, ts, [r for r, _ in rts])
    for s0, (r, t) in zip(starts, rts):
        assert (r.numel() + 255) // 256 == 32000
        _check_call(tgl, cfg, g, go, r, t, s0)


def test_batch_views_equal_per_batch_calls(tgl):
    """A training loop samples many batches per call (epoch mode) and consumes per-batch views
    (Block.batch): each view equals the per-batch call of that batch (R#7 keys)."""
    cfg = C.CONFIGS["C1"]
    src, dst, ts = C.edges("C1", cfg, device="cuda")
    g = tgl.build(src, dst, ts, n_nodes=cfg.n_nodes, add_reverse=True)
    B, M, s0 = cfg.batch, 50, 600 * 100
    r, t = C.roots(cfg, src, dst, ts, s0, M * B)
    many = tgl.Sampler(g, M * B, cfg.fanouts).run(r, t, seed=cfg.sampler_seed, root_key_base=s0)[0]
    one = tgl.Sampler(g, B, cfg.fanouts)
    for b in (0, 17, M - 1):
        got = many.batch(b * B, (b + 1) * B)
        want = one.run(r[b * B:(b + 1) * B], t[b * B:(b + 1) * B], seed=cfg.sampler_seed,
                       root_key_base=s0 + b * B)[0].trimmed()
        for x, y in zip(got[:4], want[:4]):
            assert torch.equal(x, y)


def test_batch_roots_equals_root_stream(tgl):
    """tgl_batch_roots (a5 root staging from positive edges + negatives, R#16) reproduces the root
    stream, for ranges starting at every position of an edge triple."""
    cfg = C.CONFIGS["C2"]
    src, dst, ts = C.edges("C2", cfg, device="cuda")
    for s0, n in ((0, 600), (3001, 4000), (3002, 1), (12345, 7777), (5, 0)):
        e0, s, d, ng, t = C.batch_edges(cfg, src, dst, ts, s0, max(n, 1))
        r, rt = tgl.batch_roots(s, d, ng, t, first_root=s0, n_roots=n)
        wr, wt = C.roots(cfg, src, dst, ts, s0, n)
        assert torch.equal(r, wr) and torch.equal(rt, wt)
