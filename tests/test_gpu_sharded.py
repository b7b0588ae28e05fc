"""Node-sharded mode on one GPU: W ranks simulated by W threads that share
the device and exchange through an in-process all-to-all; every rank's blocks must equal the
replicated mode's blocks bit for bit (same roots, same global root keys)."""
import math
import threading

import numpy as np
import pytest
import torch

from synth.tiny import random_graph, random_roots

pytestmark = pytest.mark.gpu


class _Hub:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.box = {}


class LocalExchange:
    def __init__(self, hub, rank):
        self.hub, self.rank, self.world = hub, rank, hub.world

    def splits(self, send_counts):
        self.hub.box[("s", self.rank)] = send_counts.cpu()
        self.hub.barrier.wait()
        recv = torch.tensor([int(self.hub.box[("s", p)][self.rank]) for p in range(self.world)], dtype=torch.int64,
                            device=send_counts.device)
        self.hub.barrier.wait()
        return recv

    def exchange(self, t, send_splits, recv_splits):
        torch.cuda.synchronize()
        self.hub.box[("x", self.rank)] = list(torch.split(t, [int(x) for x in send_splits]))
        self.hub.barrier.wait()
        out = torch.cat([self.hub.box[("x", p)][self.rank] for p in range(self.world)])
        torch.cuda.synchronize()
        self.hub.barrier.wait()
        return out


@pytest.mark.parametrize("world,strategy,S,t_s", [(2, "most_recent", 3, 5.0), (3, "uniform", 1, math.inf),
                                                  (4, "most_recent", 1, math.inf), (5, "uniform", 2, 7.0)])
def test_node_sharded_equals_replicated(world, strategy, S, t_s):
    import paper_2203_14883_b200 as tgl
    from paper_2203_14883_b200 import sharded as sh
    n_nodes = 3000
    src, dst, ts, _ = random_graph(world, n_nodes, 60_000, integer_times=True, t_max=200)
    g = tgl.build(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), torch.from_numpy(ts).cuda(),
                  n_nodes=n_nodes, add_reverse=True)
    splits = sh.edge_balanced_splits(g.indptr, world)
    assert int(splits[0]) == 0 and int(splits[-1]) == n_nodes
    shards = [sh.slice_shard(g, int(splits[r]), int(splits[r + 1])) for r in range(world)]
    roots = []
    for r in range(world):
        rn, rt = random_roots(100 + r, n_nodes, 1500 + 37 * r, integer_times=True, t_max=200)
        roots.append((torch.from_numpy(rn).cuda(), torch.from_numpy(rt).cuda(), 10_000 * r))
    hub = _Hub(world)
    results, errors = [None] * world, []

    def rank_main(r):
        try:
            ops = sh.CudaOps(shards[r], 10, strategy, S, t_s, max_roots=sum(x[0].numel() for x in roots))
            smp = sh.NodeShardedSampler(splits, LocalExchange(hub, r), ops, S, seed=7)
            results[r] = smp.run(*roots[r])
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append(e)
            hub.barrier.abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for r in range(world):
        rn, rt, base = roots[r]
        ref = tgl.sample(g, rn, rt, fanouts=[10], strategy=strategy, n_snapshots=S, snapshot_len=t_s, seed=7,
                         root_key_base=base)
        for s in range(S):
            off, nbr, eid, dt, _ = ref[s].trimmed()
            got = results[r][s]
            assert torch.equal(got.offsets, off)
            assert torch.equal(got.nbr, nbr) and torch.equal(got.eid, eid)
            assert torch.equal(got.dt.view(torch.int32), dt.view(torch.int32))


def _run_ranks(world, fn):
    hub = _Hub(world)
    errors = []

    def main(r):
        try:
            fn(r, LocalExchange(hub, r))
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append(e)
            hub.barrier.abort()

    th = [threading.Thread(target=main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("world,K", [(2, 1), (3, 3), (4, 10)])
def test_sharded_node_tables_gather_and_state_write(world, K):
    """node tables sharded by node range.  gather == the full tables' rows;
    state_write == the oracle's sequential state write of all ranks' events in (rank, index) order."""
    import oracle
    from paper_2203_14883_b200 import sharded as sh
    rng = np.random.default_rng(world * 10 + K)
    V, w = 2500, 37
    splits = torch.tensor(sorted({0, V, *rng.integers(1, V, world - 1).tolist()}), dtype=torch.int64).cuda()
    if splits.numel() != world + 1:
        splits = torch.linspace(0, V, world + 1).round().to(torch.int64).cuda()
    full = rng.standard_normal((V * K, w)).astype(np.float32)
    full_ts = rng.random(V * K).astype(np.float32)
    full_pos = rng.integers(0, K, V).astype(np.int32)
    sp = splits.cpu().numpy()
    local = [(torch.from_numpy(full[sp[r] * K:sp[r + 1] * K].copy()).cuda(),
              torch.from_numpy(full_ts[sp[r] * K:sp[r + 1] * K].copy()).cuda(),
              torch.from_numpy(full_pos[sp[r]:sp[r + 1]].copy()).cuda()) for r in range(world)]
    q_ids = [rng.integers(-1, V, int(rng.integers(0, 3000))).astype(np.int32) for _ in range(world)]
    ev = []
    for r in range(world):
        n = int(rng.integers(0, 4000))
        ev.append(((rng.zipf(1.4, n) % V).astype(np.int32), np.sort(rng.random(n)).astype(np.float32),
                   rng.standard_normal((n, w)).astype(np.float32)))
    got = [None] * world

    def fn(r, ex):
        t, tts, pos = local[r]
        tabs = sh.ShardedNodeTables(splits, ex, sh.CudaTableOps(), [t, tts], K=K, pos=pos if K > 1 else None,
                                    ts_table=None)
        got[r] = [x.cpu().numpy() for x in tabs.gather(torch.from_numpy(q_ids[r]).cuda())]
        ids, ts, rows = ev[r]
        tabs.state_write(torch.from_numpy(ids).cuda(), torch.from_numpy(ts).cuda(),
                         [torch.from_numpy(rows).cuda(), torch.from_numpy(ts).cuda()])

    _run_ranks(world, fn)
    node_rows, node_ts = full.reshape(V, K * w), full_ts.reshape(V, K)
    for r in range(world):
        ids = q_ids[r]
        want = np.where((ids >= 0)[:, None], node_rows[np.clip(ids, 0, V - 1)], 0.0)
        np.testing.assert_array_equal(got[r][0], want)
        np.testing.assert_array_equal(got[r][1].reshape(len(ids), K), np.where((ids >= 0)[:, None], node_ts[np.clip(ids, 0, V - 1)], 0.0))
    # reference: one sequential state write of every rank's events in (rank, index) order
    ids = np.concatenate([e[0] for e in ev])
    ts = np.concatenate([e[1] for e in ev])
    rows = np.concatenate([e[2] for e in ev])
    ref, ref_ts, ref_pos = full.copy(), full_ts.copy(), full_pos.copy()
    oracle.state_write(ids, ts, n_nodes=V, K=K, tables=[(rows, ref), (ts.copy(), ref_ts)],
                       pos=ref_pos if K > 1 else None)
    for r in range(world):
        t, tts, pos = local[r]
        np.testing.assert_array_equal(t.cpu().numpy(), ref[sp[r] * K:sp[r + 1] * K])
        np.testing.assert_array_equal(tts.cpu().numpy(), ref_ts[sp[r] * K:sp[r + 1] * K])
        if K > 1:
            np.testing.assert_array_equal(pos.cpu().numpy(), ref_pos[sp[r]:sp[r + 1]])
