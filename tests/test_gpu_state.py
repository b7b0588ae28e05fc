"""GPU parity of tgl_state_write (Fig. 2 step 6, R#25) against the CPU oracle, bit for bit: node
memory (K = 1, last event wins) and mailbox rings (K > 1, K most recent in cursor order), several
tables of different widths and alignments in one call, Zipf hubs (a node with far more than K
events in a batch), multi-tile batches, out-of-range ids (skipped + sticky ERANGE), n = 0."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tgl():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    import paper_2203_14883_b200 as m
    return m


def _case(rng, V, n, K, widths, bad=False):
    ids = (rng.zipf(1.3, n) % V).astype(np.int32)
    if bad and n:
        ids[rng.integers(0, n, max(1, n // 50))] = rng.choice([-1, V, V + 7])
    ts = np.sort(rng.integers(0, 10**6, n)).astype(np.float32)
    rows = [rng.integers(-2**31, 2**31 - 1, (n, w // 4), dtype=np.int64).astype(np.int32) if w % 4 == 0
            else rng.integers(0, 255, (n, w), dtype=np.int64).astype(np.uint8) for w in widths]
    tables = [rng.integers(-2**31, 2**31 - 1, (V * K, w // 4), dtype=np.int64).astype(np.int32) if w % 4 == 0
              else rng.integers(0, 255, (V * K, w), dtype=np.int64).astype(np.uint8) for w in widths]
    pos = rng.integers(0, K, V).astype(np.int32)
    tts = rng.random(V * K).astype(np.float32)
    return ids, ts, rows, tables, pos, tts


@pytest.mark.parametrize("V,n,K,widths", [(50, 600, 1, [400, 4, 1712]), (1000, 20000, 1, [400, 4]),
                                          (37, 5000, 3, [12, 400]), (2000, 9000, 10, [1712, 4]),
                                          (7, 100, 4, [3, 16, 6]), (100000, 50000, 2, [64])])
def test_state_write_bit_exact(tgl, V, n, K, widths):
    rng = np.random.default_rng(V + n + K)
    for bad in (False, True):
        ids, ts, rows, tables, pos, tts = _case(rng, V, n, K, widths, bad)
        g_tables = [torch.from_numpy(t.copy()).cuda() for t in tables]
        g_rows = [torch.from_numpy(r).cuda() for r in rows]
        g_pos = torch.from_numpy(pos.copy()).cuda()
        g_tts = torch.from_numpy(tts.copy()).cuda()
        tgl.state_write(torch.from_numpy(ids).cuda(), torch.from_numpy(ts).cuda(), list(zip(g_rows, g_tables)),
                        n_nodes=V, K=K, pos=g_pos if K > 1 else None, ts_table=g_tts)
        code = tgl.check(None)
        o_pos = pos.copy()
        want = oracle.state_write(ids, ts, n_nodes=V, K=K, tables=list(zip(rows, tables)),
                                  pos=o_pos if K > 1 else None, ts_table=tts)
        assert code == want
        for gt, t in zip(g_tables, tables):
            np.testing.assert_array_equal(gt.cpu().numpy(), t)
        np.testing.assert_array_equal(g_tts.cpu().numpy().view(np.uint32), tts.view(np.uint32))
        if K > 1:
            np.testing.assert_array_equal(g_pos.cpu().numpy(), o_pos)


def test_state_write_empty_and_errors(tgl):
    from paper_2203_14883_b200 import _lib
    t = torch.zeros(10, 4, dtype=torch.float32, device="cuda")
    tgl.state_write(torch.zeros(0, dtype=torch.int32, device="cuda"), None,
                    [(torch.zeros(0, 4, device="cuda"), t)], n_nodes=10)
    assert tgl.check(None) == 0 and int(t.abs().sum().item()) == 0
    L_ = _lib.load()
    ids = torch.zeros(3, dtype=torch.int32, device="cuda")
    ws = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    assert L_.tgl_state_write(ids.data_ptr(), None, 3, 10, 0, None, None, None, 0, ws.data_ptr(), 1 << 20, None) == -1
    assert L_.tgl_state_write(ids.data_ptr(), None, 3, 10, 4, None, None, None, 0, ws.data_ptr(), 1 << 20, None) == -1
    assert L_.tgl_state_write(ids.data_ptr(), None, 3, 10, 1, None, None, None, 0, ws.data_ptr(), 16, None) == -5


def test_chunk_schedule_equals_oracle(tgl):
    """tgl_chunk_schedule (Alg. 2, R#26) vs the oracle's schedule, over epochs and shapes."""
    for n, bs, cs in [(157_474, 600, 100), (1_000_000, 4000, 250), (599, 600, 100), (0, 8, 2), (10_000, 600, 600)]:
        for epoch in (0, 1, 2, 77, 2**33 + 5):
            first, nb = tgl.chunk_schedule(n, bs, cs, epoch, seed=42)
            want = oracle.chunk_schedule(n, bs, cs, epoch, seed=42)
            k = int(nb.item())
            assert k == len(want)
            np.testing.assert_array_equal(first[:k].cpu().numpy(), np.array(want, dtype=np.int64))


def test_fused_gather_equals_separate_gathers():
    """tgl_fused_gather (the copy kernel writes the rows of each output's node / edge) equals
    tgl_gather over the block's nbr / eid, byte for byte -- C3's tables (100- and 428-float rows,
    1-float timestamps, 128-float edge features), most_recent 1 layer and uniform 2 layers."""
    import paper_2203_14883_b200 as tgl
    from synth import configs as C
    cfg = C.CONFIGS["C3"]
    src, dst, ts = C.edges("C3", cfg, device="cuda")
    g = tgl.build(src, dst, ts, n_nodes=cfg.n_nodes, add_reverse=True)
    tabs = C.tables(cfg, device="cuda")
    r, t = C.roots(cfg, src, dst, ts, 600 * 2000, 600 * 40)
    spec = [(tabs["memory"], "node"), (tabs["mem_ts"], "node"), (tabs["mailbox"], "node"),
            (tabs["edge_feat"], "edge")]
    for fan, strat in (([10], "most_recent"), ([5, 4], "uniform")):
        smp = tgl.Sampler(g, r.numel(), fan, strat, fused_gather=spec)
        blocks = smp.run(r, t, seed=3, root_key_base=600 * 2000)
        last = blocks[-1]
        n = int(last.nnz_dev.item())
        for (tab, by), got in zip(spec, smp.fused_outs):
            want = tgl.gather(last.nbr if by == "node" else last.eid, [tab], n_ids_dev=last.nnz_dev)[0]
            assert torch.equal(got[:n], want[:n])
        assert tgl.check(g) == 0
