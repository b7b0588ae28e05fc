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
