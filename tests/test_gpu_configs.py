"""GPU parity on the five paper-shaped workloads (BASELINE.json configs C1-C5) at FULL size.

Inputs: synth.configs (seeded generators, generated on the GPU -- integer-only, so identical to a
CPU generation).  Expected values: oracle/ only.  The CUDA side runs in the launch configuration
bench.py times (many batches per tgl_sample call, root_key_base = global root index); the oracle
runs per batch.  C1-C3: the whole T-CSR is compared; C1 the whole epoch of roots.  C4: the oracle
builds the full 191 M-edge T-CSR on the host; sampled batches spread over the epoch are compared.
C5 (1.3 B edges): the oracle builds the T-CSR restricted to the sampled roots' nodes (oracle's own
count/fill passes over the stream sub-selected to those nodes); sampled batches are compared.
Every comparison is bit-exact; full-size properties (no leak, counts <= k) are checked on the
whole GPU output.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from synth import configs as C

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tgl():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_2203_14883_b200 as m
    return m


def _strategy(cfg):
    return 0 if cfg.strategy == "most_recent" else 1


def _spread_batches(cfg, n_windows, per_window):
    """Batch indices: n_windows windows of consecutive batches, evenly spread over the epoch."""
    n_batches = cfg.n_roots_epoch // cfg.batch
    starts = np.linspace(0, n_batches - per_window, n_windows).astype(np.int64)
    return [int(s + j) for s in starts for j in range(per_window)]


def _compare_call(tgl, cfg, g_gpu, g_orc, src, dst, ts, batches):
    """One GPU call over all `batches` (concatenated roots), oracle per batch; bit-exact."""
    B = cfg.batch
    rs, rts, bases = [], [], []
    for b in batches:
        r, t = C.roots(cfg, src, dst, ts, b * B, B)
        rs.append(r)
        rts.append(t)
        bases.append(b * B)
    L, S = len(cfg.fanouts), cfg.n_snapshots
    # the GPU call covers consecutive runs of batches; split into runs of consecutive batch ids
    runs, cur = [], [0]
    for j in range(1, len(batches)):
        if batches[j] == batches[j - 1] + 1:
            cur.append(j)
        else:
            runs.append(cur)
            cur = [j]
    runs.append(cur)
    for run in runs:
        R = torch.cat([rs[j] for j in run])
        T = torch.cat([rts[j] for j in run])
        blocks = tgl.sample(g_gpu, R, T, fanouts=cfg.fanouts, strategy=cfg.strategy, n_snapshots=S,
                            snapshot_len=cfg.snapshot_len, seed=cfg.sampler_seed, root_key_base=bases[run[0]])
        got = [[x.cpu().numpy() for x in b.trimmed()[:4]] for b in blocks]
        # full-size properties on the GPU output
        for (off, nbr, eid, dt) in got:
            assert np.all(dt > 0), "leak: sampled edge not strictly earlier than its root (P:L267)"
            assert np.all(np.diff(off) >= 0)
        for li in range(L):
            for s in range(S):
                off = got[li * S + s][0]
                assert np.all(np.diff(off) <= cfg.fanouts[li])
        # oracle per batch, then compare block by block (layer 0 roots split per batch; deeper
        # layers' roots follow their batch's layer-0 outputs)
        root_off = {li * S + s: 0 for li in range(L) for s in range(S)}
        edge_off = {li * S + s: 0 for li in range(L) for s in range(S)}
        for j in run:
            bo = oracle.sample(g_orc, rs[j].cpu().numpy(), rts[j].cpu().numpy(), fanouts=cfg.fanouts,
                               strategy=_strategy(cfg), n_snapshots=S, snapshot_len=cfg.snapshot_len,
                               seed=cfg.sampler_seed, root_key_base=bases[j])
            for q, o in enumerate(bo):
                n = len(o["offsets"]) - 1
                nnz = len(o["nbr"])
                off, nbr, eid, dt = got[q]
                r0, e0 = root_off[q], edge_off[q]
                np.testing.assert_array_equal(off[r0:r0 + n + 1] - off[r0], o["offsets"], err_msg=f"batch {batches[j]}")
                assert off[r0] == e0
                np.testing.assert_array_equal(nbr[e0:e0 + nnz], o["nbr"])
                np.testing.assert_array_equal(eid[e0:e0 + nnz], o["eid"])
                np.testing.assert_array_equal(dt[e0:e0 + nnz].view(np.uint32), o["dt"].view(np.uint32))
                root_off[q] += n
                edge_off[q] += nnz
        for q in range(L * S):
            assert root_off[q] == len(got[q][0]) - 1 and edge_off[q] == len(got[q][1])


@pytest.mark.parametrize("key", ["C1", "C2", "C3", "C6"])
def test_small_configs_full_tcsr_and_batches(tgl, key):
    cfg = C.CONFIGS[key]
    src, dst, ts = C.edges(key, cfg, device="cuda")
    g = tgl.build(src, dst, ts, n_nodes=cfg.n_nodes, add_reverse=cfg.add_reverse)
    go = oracle.build(src.cpu().numpy(), dst.cpu().numpy(), ts.cpu().numpy(), n_nodes=cfg.n_nodes,
                      add_reverse=cfg.add_reverse)
    for name in ("indptr", "nbr", "ts", "eid"):
        np.testing.assert_array_equal(getattr(g, name).cpu().numpy().view(go[name].dtype), go[name], err_msg=name)
    if key == "C1":   # the whole epoch in one call, the way bench.py runs it
        batches = list(range(cfg.n_roots_epoch // cfg.batch))
    else:
        batches = _spread_batches(cfg, 8, 8)
    _compare_call(tgl, cfg, g, go, src, dst, ts, batches)


def test_c3_gather_bit_exact(tgl):
    """C3 (TGN/JODIE path): gather node memory, mem_ts, mailbox (428-wide), mail_ts by the sampled
    node ids and edge features by the sampled eids (Fig. 2 step 2), vs the oracle."""
    cfg = C.CONFIGS["C3"]
    src, dst, ts = C.edges("C3", cfg, device="cuda")
    g = tgl.build(src, dst, ts, n_nodes=cfg.n_nodes, add_reverse=True)
    tabs = C.tables(cfg, device="cuda")
    r, t = C.roots(cfg, src, dst, ts, 600 * 3000, 600 * 16)
    blocks = tgl.sample(g, r, t, fanouts=[10], seed=cfg.sampler_seed, root_key_base=600 * 3000)
    b = blocks[0]
    node_tables = [tabs["memory"], tabs["mem_ts"], tabs["mailbox"], tabs["mail_ts"]]
    outs = tgl.gather(b.nbr, node_tables, n_ids_dev=b.nnz_dev)
    outs_r = tgl.gather(r, node_tables)
    oute = tgl.gather(b.eid, [tabs["edge_feat"]], n_ids_dev=b.nnz_dev)[0]
    assert tgl.check(None) == 0
    nnz = int(b.nnz_dev.item())
    ids = b.nbr[:nnz].cpu().numpy()
    for tab, out in zip(node_tables, outs):
        want, err = oracle.gather(ids, tab.cpu().numpy())
        assert err == 0
        np.testing.assert_array_equal(out[:nnz].cpu().numpy().view(np.uint8), want.view(np.uint8))
    for tab, out in zip(node_tables, outs_r):
        want, _ = oracle.gather(r.cpu().numpy(), tab.cpu().numpy())
        np.testing.assert_array_equal(out.cpu().numpy().view(np.uint8), want.view(np.uint8))
    want, _ = oracle.gather(b.eid[:nnz].cpu().numpy(), tabs["edge_feat"].cpu().numpy())
    np.testing.assert_array_equal(oute[:nnz].cpu().numpy().view(np.uint8), want.view(np.uint8))


def test_c4_gdelt_full_size(tgl):
    cfg = C.CONFIGS["C4"]
    src, dst, ts = C.edges("C4", cfg, device="cuda")
    g = tgl.build(src, dst, ts, n_nodes=cfg.n_nodes, add_reverse=False)
    go = oracle.build(src.cpu().numpy(), dst.cpu().numpy(), ts.cpu().numpy(), n_nodes=cfg.n_nodes,
                      add_reverse=False)
    np.testing.assert_array_equal(g.indptr.cpu().numpy(), go["indptr"])
    # full T-CSR arrays compared on a stride (2.3 GB each on the host)
    for name in ("nbr", "ts", "eid"):
        a = getattr(g, name)[::997].cpu().numpy().view(go[name].dtype)
        np.testing.assert_array_equal(a, go[name][::997], err_msg=name)
    _compare_call(tgl, cfg, g, go, src, dst, ts, _spread_batches(cfg, 4, 4))


def test_c5_mag_full_size(tgl):
    cfg = C.CONFIGS["C5"]
    src, dst, ts = C.edges("C5", cfg, device="cuda")
    g = tgl.build(src, dst, ts, n_nodes=cfg.n_nodes, add_reverse=True)
    assert int(g.indptr[-1].item()) == 2 * cfg.n_edges
    batches = _spread_batches(cfg, 8, 4)
    nodes = torch.cat([C.roots(cfg, src, dst, ts, b * cfg.batch, cfg.batch)[0] for b in batches])
    s_np, d_np, t_np, e_np, keep = C.relevant_substream(src, dst, ts, nodes, cfg.n_nodes, True)
    go = oracle.build_restricted(lambda: iter([(s_np, d_np, t_np, e_np, 0)]), n_nodes=cfg.n_nodes,
                                 add_reverse=True, keep=keep)
    # the restricted oracle lists equal the GPU T-CSR lists of the kept nodes
    some = np.unique(nodes.cpu().numpy())[:: max(1, len(np.unique(nodes.cpu().numpy())) // 200)]
    for v in some:
        lo, hi = int(go["indptr"][v]), int(go["indptr"][v + 1])
        glo, ghi = int(g.indptr[v].item()), int(g.indptr[v + 1].item())
        assert hi - lo == ghi - glo
        np.testing.assert_array_equal(g.eid[glo:ghi].cpu().numpy(), go["eid"][lo:hi])
    _compare_call(tgl, cfg, g, go, src, dst, ts, batches)


def test_c5_tcsr_full_digest(tgl):
    """The WHOLE C5 T-CSR (121 M lists, 2.6 B slots) against the oracle's build, by digest: the
    node range is cut into 8 parts; per part the oracle builds the lists of its nodes with its own
    count / fill passes over the stream sub-selected to them (build_restricted), and 64 sub-ranges
    per part are compared through tgl_block_digest over (indptr, nbr, eid, ts) -- FNV-1a of every
    list element, so any difference anywhere in the 31 GB of lists fails."""
    cfg = C.CONFIGS["C5"]
    src, dst, ts = C.edges("C5", cfg, device="cuda")
    g = tgl.build(src, dst, ts, n_nodes=cfg.n_nodes, add_reverse=True)
    as_block = tgl.Block(offsets=g.indptr, nbr=g.nbr, eid=g.eid, dt=g.ts, ts_edge=None, n_roots_dev=None,
                         nnz_dev=None)
    V, parts, sub = cfg.n_nodes, 8, 64
    for p in range(parts):
        lo, hi = V * p // parts, V * (p + 1) // parts
        nodes = torch.arange(lo, hi, dtype=torch.int32, device="cuda")
        s_np, d_np, t_np, e_np, keep = C.relevant_substream(src, dst, ts, nodes, V, True)
        go = oracle.build_restricted(lambda: iter([(s_np, d_np, t_np, e_np, 0)]), n_nodes=V, add_reverse=True, keep=keep)
        del s_np, d_np, t_np, e_np
        bounds = [lo + (hi - lo) * q // sub for q in range(sub + 1)]
        gd = tgl.block_digest(as_block, torch.tensor(bounds, dtype=torch.int64, device="cuda")).cpu().numpy()
        ip = go["indptr"]
        od = []
        for q in range(sub):
            a, b = bounds[q], bounds[q + 1]
            e0, e1 = int(ip[a]), int(ip[b])
            od.append(oracle.block_digest({"offsets": ip[a:b + 1], "nbr": go["nbr"][e0:e1], "eid": go["eid"][e0:e1],
                                           "dt": go["ts"][e0:e1]}))
        np.testing.assert_array_equal(gd.view(np.uint64), np.array(od, dtype=np.uint64), err_msg=f"part {p}")
        # the restricted oracle's indptr differences equal the GPU degrees on this part
        np.testing.assert_array_equal(np.diff(ip[lo:hi + 1]), torch.diff(g.indptr[lo:hi + 1]).cpu().numpy())
        del go
