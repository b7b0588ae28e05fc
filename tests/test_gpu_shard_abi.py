"""Node-sharded mode behind the C ABI (SURVEY 8(b) tgl_shard_create / tgl_sample_sharded, 8(e)).

* tgl_tcsr_build_range: every rank builds only its node range; the range's lists equal the full
  build's lists (which are oracle-pinned elsewhere) element for element, and tgl_tcsr_indptr equals
  the full build's indptr.
* tgl_sample_sharded over W ranks (an in-process group: W threads on this GPU, exchanging by device
  copies; and NCCL with a 1-rank communicator): every rank's blocks equal, bit for bit, what the
  replicated tgl_sample writes for the same roots and key base -- which the oracle pins
  (tests/test_gpu_parity.py) -- over 1-3 layers, S = 1 and 3 snapshots (finite windows inherited
  by deeper layers, R#3), both strategies.  One check also goes to the oracle directly.
"""
import math
import threading

import numpy as np
import pytest
import torch

import oracle
from synth import configs as C
from synth.tiny import random_graph, random_roots

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tgl():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_2203_14883_b200 as m
    return m


def splits_of(indptr, world):
    from paper_2203_14883_b200.sharded import edge_balanced_splits
    return [int(x) for x in edge_balanced_splits(indptr, world).cpu()]


def build_ranges(tgl, src, dst, ts, n_nodes, add_rev, world):
    indptr = tgl.tcsr_indptr(src, dst, ts, n_nodes=n_nodes, add_reverse=add_rev)
    sp = splits_of(indptr, world)
    shards = [tgl.build_range(src, dst, ts, n_nodes=n_nodes, add_reverse=add_rev, node_lo=sp[r], node_hi=sp[r + 1],
                              n_local_stored=int(indptr[sp[r + 1]] - indptr[sp[r]])) for r in range(world)]
    return indptr, sp, shards


def blocks_np(blocks):
    out = []
    for b in blocks:
        off, nbr, eid, dt, te = b.trimmed()
        out.append([x.cpu().numpy().copy() for x in (off, nbr, eid, dt.view(torch.int32))]
                   + ([] if te is None else [te.view(torch.int32).cpu().numpy().copy()]))
    return out


def assert_same(a, b, what):
    assert len(a) == len(b)
    for q, (x, y) in enumerate(zip(a, b)):
        for j, (u, v) in enumerate(zip(x, y)):
            np.testing.assert_array_equal(u, v, err_msg=f"{what}: block {q} array {j}")


def run_sharded(tgl, shards, sp, per_rank, fanouts, strategy, S, t_s, seed, nccl=False):
    """per_rank: [(roots, root_ts, key_base)] -> per rank the blocks (numpy) and the stats."""
    W = len(shards)
    grp = None if nccl else tgl.ShardGroup(W)
    uid = tgl.nccl_id() if nccl else None
    smps = [tgl.ShardSampler(shards[r], sp, r, W, max(per_rank[r][0].numel(), 1), fanouts, strategy, S, t_s,
                             nccl_id=uid, group=grp) for r in range(W)]
    res, errs = [None] * W, []

    def work(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                rr, tt, base = per_rank[r]
                bl = smps[r].run(rr, tt, seed=seed, root_key_base=base)
                st.synchronize()
                res[r] = blocks_np(bl)
        except Exception as e:  # noqa: BLE001
            errs.append(e)
    th = [threading.Thread(target=work, args=(r,)) for r in range(W)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    stats = [s.stats() for s in smps]
    for s in shards:
        assert tgl.check(s) == 0
    return res, stats


def test_build_range_equals_full_build(tgl):
    for case, (V, E, rev, W) in enumerate([(300, 4000, True, 3), (50, 2000, False, 4), (1, 10, True, 1),
                                           (400, 0, True, 2)]):
        src, dst, ts, _ = random_graph(case + 900, V, E, with_eid=False, integer_times=True)
        s, d, t = (torch.as_tensor(x).cuda() for x in (src, dst, ts))
        g = tgl.build(s, d, t, n_nodes=V, add_reverse=rev)
        indptr, sp, shards = build_ranges(tgl, s, d, t, V, rev, W)
        np.testing.assert_array_equal(indptr.cpu().numpy(), g.indptr.cpu().numpy())
        for r, sh in enumerate(shards):
            lo, hi = sp[r], sp[r + 1]
            a, b = int(g.indptr[lo]), int(g.indptr[hi])
            np.testing.assert_array_equal(sh.indptr.cpu().numpy(), (g.indptr[lo:hi + 1] - a).cpu().numpy())
            for name in ("nbr", "ts", "eid"):
                np.testing.assert_array_equal(getattr(sh, name).cpu().numpy(), getattr(g, name)[a:b].cpu().numpy())


CASES = [  # fanouts, strategy, S, t_s
    ([10], "most_recent", 3, 5.0),
    ([10, 10], "uniform", 1, math.inf),
    ([5, 4], "most_recent", 3, 40.0),
    ([3, 3, 2], "uniform", 2, 30.0),
]


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_sharded_equals_replicated(tgl, world, case):
    fanouts, strategy, S, t_s = CASES[case]
    V, E = 700, 30000
    src, dst, ts, _ = random_graph(4242 + case, V, E, with_eid=False, integer_times=True)
    s, d, t = (torch.as_tensor(x).cuda() for x in (src, dst, ts))
    g = tgl.build(s, d, t, n_nodes=V, add_reverse=True)
    _, sp, shards = build_ranges(tgl, s, d, t, V, True, world)
    per_rank = []
    for r in range(world):
        n = [500, 1300, 0, 777][r % 4] if world > 1 else 2000
        rr, tt = random_roots(77 + r, V, n, integer_times=True)
        per_rank.append((torch.as_tensor(rr).cuda(), torch.as_tensor(tt).cuda(), 10_000 * r))
    got, stats = run_sharded(tgl, shards, sp, per_rank, fanouts, strategy, S, t_s, seed=5)
    for r in range(world):
        rr, tt, base = per_rank[r]
        want = tgl.sample(g, rr, tt, fanouts=fanouts, strategy=strategy, n_snapshots=S, snapshot_len=t_s, seed=5,
                          root_key_base=base)
        assert_same(got[r], blocks_np(want), f"world {world} rank {r}")
    if world > 1:
        assert sum(x["bytes_sent"] for x in stats) == sum(x["bytes_recv"] for x in stats) > 0
    assert all(x["host_syncs"] == 2 * (1 + (len(fanouts) - 1) * S) for x in stats)


def test_sharded_against_oracle_and_nccl(tgl):
    """NCCL transport (1-rank communicator) on a scaled C5 (1 layer, 3 snapshots of 5) straight
    against the oracle, and the 4-rank in-process group on the same roots."""
    cfg = C.scaled(C.CONFIGS["C5"], 200_000, 2_000_000)
    src, dst, ts = C.edges("C5", cfg, device="cuda")
    r, t = C.roots(cfg, src, dst, ts, 3_000_000, 40_000)
    go = oracle.build(src.cpu().numpy(), dst.cpu().numpy(), ts.cpu().numpy(), n_nodes=cfg.n_nodes, add_reverse=True)
    want = oracle.sample(go, r.cpu().numpy(), t.cpu().numpy(), fanouts=cfg.fanouts, strategy=0,
                         n_snapshots=cfg.n_snapshots, snapshot_len=cfg.snapshot_len, seed=cfg.sampler_seed,
                         root_key_base=3_000_000)
    want_np = [[o["offsets"], o["nbr"], o["eid"], o["dt"].view(np.int32)] for o in want]
    _, sp, shards = build_ranges(tgl, src, dst, ts, cfg.n_nodes, True, 1)
    got, _ = run_sharded(tgl, shards, sp, [(r, t, 3_000_000)], cfg.fanouts, cfg.strategy, cfg.n_snapshots,
                         cfg.snapshot_len, cfg.sampler_seed, nccl=True)
    assert_same(got[0], want_np, "nccl world 1")
    W = 4
    _, sp, shards = build_ranges(tgl, src, dst, ts, cfg.n_nodes, True, W)
    q = r.numel() // W
    per_rank = [(r[i * q:(i + 1) * q], t[i * q:(i + 1) * q], 3_000_000 + i * q) for i in range(W)]
    got, stats = run_sharded(tgl, shards, sp, per_rank, cfg.fanouts, cfg.strategy, cfg.n_snapshots,
                             cfg.snapshot_len, cfg.sampler_seed)
    # stitch the ranks' blocks back together and compare with the oracle's single call
    for b in range(cfg.n_snapshots):
        off = np.concatenate([[0]] + [got[i][b][0][1:] + sum(int(got[j][b][0][-1]) for j in range(i))
                                      for i in range(W)])
        np.testing.assert_array_equal(off, want_np[b][0])
        for j in (1, 2, 3):
            np.testing.assert_array_equal(np.concatenate([got[i][b][j] for i in range(W)]), want_np[b][j])


@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_node_state(tgl, world):
    """tgl_shard_gather / tgl_shard_state_write over W ranks on threads: the
    gathered rows equal the full tables' rows, and the owners' local tables after the write equal
    the oracle's sequential write (R#25) of all ranks' events in (rank, index) order."""
    V, E, K, dm, dmail = 500, 20000, 3, 7, 5
    src, dst, ts, _ = random_graph(31, V, E, with_eid=False, integer_times=True)
    s, d, t = (torch.as_tensor(x).cuda() for x in (src, dst, ts))
    _, sp, shards = build_ranges(tgl, s, d, t, V, True, world)
    grp = tgl.ShardGroup(world)
    smps = [tgl.ShardSampler(shards[r], sp, r, world, 1, [1], group=grp) for r in range(world)]
    rng = np.random.default_rng(5)
    mem = torch.as_tensor(rng.standard_normal((V, dm)).astype(np.float32)).cuda()
    mail = torch.as_tensor(rng.standard_normal((V, K, dmail)).astype(np.float32)).cuda()
    pos = torch.as_tensor(rng.integers(0, K, V).astype(np.int32)).cuda()
    mts = torch.zeros(V * K, dtype=torch.float32, device="cuda")
    loc = [dict(mem=mem[sp[r]:sp[r + 1]].clone(), mail=mail[sp[r]:sp[r + 1]].clone(), pos=pos[sp[r]:sp[r + 1]].clone(),
                mts=mts[sp[r] * K:sp[r + 1] * K].clone()) for r in range(world)]
    ids = [torch.as_tensor(np.where(rng.random(n) < 0.1, -1, rng.integers(0, V, n)).astype(np.int32)).cuda()
           for n in (900, 0, 1500)[:world]]
    ev = [torch.as_tensor(rng.integers(0, V, n).astype(np.int32)).cuda() for n in (800, 1200, 0)[:world]]
    ev_t = [torch.sort(torch.as_tensor(rng.random(x.numel()).astype(np.float32) * 100).cuda())[0] for x in ev]
    ev_mem = [torch.as_tensor(rng.standard_normal((x.numel(), dm)).astype(np.float32)).cuda() for x in ev]
    ev_mail = [torch.as_tensor(rng.standard_normal((x.numel(), dmail)).astype(np.float32)).cuda() for x in ev]
    got, errs = [None] * world, []

    def work(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                g_mem, g_mail = smps[r].gather(ids[r], [loc[r]["mem"], loc[r]["mail"]])
                st.synchronize()
                got[r] = (g_mem.cpu().numpy(), g_mail.cpu().numpy())
                smps[r].state_write(ev[r], ev_t[r], [(ev_mem[r], loc[r]["mem"])], K=1)
                smps[r].state_write(ev[r], ev_t[r], [(ev_mail[r], loc[r]["mail"])], K=K, pos=loc[r]["pos"],
                                    ts_table=loc[r]["mts"])
                st.synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(e)
    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=600)
    assert not errs, errs
    assert tgl.check(None) == 0
    full_mem, full_mail = mem.cpu().numpy(), mail.cpu().numpy()
    for r in range(world):
        idn = ids[r].cpu().numpy()
        want_mem = np.where((idn >= 0)[:, None], full_mem[np.maximum(idn, 0)], 0)
        want_mail = np.where((idn >= 0)[:, None, None], full_mail[np.maximum(idn, 0)], 0)
        np.testing.assert_array_equal(got[r][0], want_mem)
        np.testing.assert_array_equal(got[r][1], want_mail)
    # oracle: all events in (rank, index) order on the full tables
    all_ids = np.concatenate([x.cpu().numpy() for x in ev])
    all_t = np.concatenate([x.cpu().numpy() for x in ev_t])
    w_mem = full_mem.copy()
    w_mail = full_mail.reshape(V * K, dmail).copy()
    w_pos, w_ts = pos.cpu().numpy().copy(), mts.cpu().numpy().copy()
    oracle.state_write(all_ids, all_t, n_nodes=V, K=1, tables=[(np.concatenate([x.cpu().numpy() for x in ev_mem]), w_mem)])
    oracle.state_write(all_ids, all_t, n_nodes=V, K=K, tables=[(np.concatenate([x.cpu().numpy() for x in ev_mail]),
                                                                w_mail)], pos=w_pos, ts_table=w_ts)
    for r in range(world):
        lo, hi = sp[r], sp[r + 1]
        np.testing.assert_array_equal(loc[r]["mem"].cpu().numpy(), w_mem[lo:hi])
        np.testing.assert_array_equal(loc[r]["mail"].cpu().numpy().reshape(-1, dmail), w_mail[lo * K:hi * K])
        np.testing.assert_array_equal(loc[r]["pos"].cpu().numpy(), w_pos[lo:hi])
        np.testing.assert_array_equal(loc[r]["mts"].cpu().numpy(), w_ts[lo * K:hi * K])
