"""Multi-process (world_size 2, gloo, CPU) test of the node-sharded exchange protocol
(paper_2203_14883_b200/sharded.py).  The CUDA ops are replaced by a CPU test double built on the
oracle (tests only); the exchange is the real torch.distributed all_to_all_single.  Each rank's
blocks must equal the oracle's replicated-mode blocks for the same roots and global keys."""
import math
import os
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]

WORKER = textwrap.dedent(r'''
    import math, os, sys
    sys.path.insert(0, os.environ["REPO"])
    import numpy as np, torch, torch.distributed as dist
    import oracle
    from synth.tiny import random_graph, random_roots
    # import the orchestration module without loading the CUDA library (CPU box)
    import importlib.util
    spec = importlib.util.spec_from_file_location("sharded", os.path.join(os.environ["REPO"], "paper_2203_14883_b200", "sharded.py"))
    sh = importlib.util.module_from_spec(spec); spec.loader.exec_module(sh)

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    S, t_s, k, strategy = int(os.environ["S"]), float(os.environ["TS"]), 10, int(os.environ["STRAT"])
    n_nodes = 400
    src, dst, ts, _ = random_graph(3, n_nodes, 8000, integer_times=True, t_max=100)
    full = oracle.build(src, dst, ts, n_nodes=n_nodes, add_reverse=True)
    splits = sh.edge_balanced_splits(torch.from_numpy(full["indptr"]), world)
    lo, hi = int(splits[rank]), int(splits[rank + 1])

    class OracleOps:   # CPU test double of CudaOps
        def bucket(self, roots, splits, world):
            owner = np.searchsorted(splits.numpy(), roots.numpy(), side="right") - 1
            perm = np.argsort(owner, kind="stable").astype(np.int32)
            return torch.from_numpy(perm), torch.from_numpy(np.bincount(owner, minlength=world).astype(np.int64))
        def pack(self, perm, roots, root_ts, keys):
            return roots[perm.long()], root_ts[perm.long()], keys[perm.long()]
        def sample(self, roots, root_ts, keys, seed):
            local = roots.numpy()
            assert np.all((local >= lo) & (local < hi)), "request routed to the wrong owner"
            out = []
            for s in range(S):
                b = oracle.sample_block(full, local, root_ts.numpy(), keys.numpy().view(np.uint64), None,
                                        layer=0, snapshot=s, snapshot_len=t_s, k=k, strategy=strategy,
                                        seed=seed, want_children=False)
                off = torch.from_numpy(b["offsets"])
                out.append((torch.from_numpy(np.diff(b["offsets"]).astype(np.int32)), torch.from_numpy(b["nbr"]),
                            torch.from_numpy(b["eid"]), torch.from_numpy(b["dt"]), off))
            return out
        def unpermute(self, perm, counts, nbr, eid, dt):
            p = perm.numpy(); c = counts.numpy().astype(np.int64)
            src_off = np.concatenate([[0], np.cumsum(c)])
            cnt_orig = np.zeros(len(p), np.int64); cnt_orig[p] = c
            off = np.concatenate([[0], np.cumsum(cnt_orig)])
            nb, ed, d = np.zeros_like(nbr.numpy()), np.zeros_like(eid.numpy()), np.zeros_like(dt.numpy())
            for j, i in enumerate(p):
                nb[off[i]:off[i+1]] = nbr.numpy()[src_off[j]:src_off[j+1]]
                ed[off[i]:off[i+1]] = eid.numpy()[src_off[j]:src_off[j+1]]
                d[off[i]:off[i+1]] = dt.numpy()[src_off[j]:src_off[j+1]]
            return torch.from_numpy(off), torch.from_numpy(nb), torch.from_numpy(ed), torch.from_numpy(d)

    rn, rt = random_roots(50 + rank, n_nodes, 300 + 17 * rank, integer_times=True, t_max=100)
    base = 1000 * rank
    smp = sh.NodeShardedSampler(splits, sh.DistExchange(), OracleOps(), S, seed=11)
    got = smp.run(torch.from_numpy(rn), torch.from_numpy(rt), base)
    ref = oracle.sample(full, rn, rt, fanouts=[k], strategy=strategy, n_snapshots=S, snapshot_len=t_s, seed=11,
                        root_key_base=base)
    for s in range(S):
        assert np.array_equal(got[s].offsets.numpy(), ref[s]["offsets"])
        assert np.array_equal(got[s].nbr.numpy(), ref[s]["nbr"])
        assert np.array_equal(got[s].eid.numpy(), ref[s]["eid"])
        assert np.array_equal(got[s].dt.numpy().view(np.uint32), ref[s]["dt"].view(np.uint32))
    dist.barrier()
    dist.destroy_process_group()
    print(f"RANK{rank}OK", flush=True)
''')


@pytest.mark.parametrize("S,ts,strat", [(3, 5.0, 0), (1, math.inf, 1)])
def test_node_sharded_protocol_gloo_world2(tmp_path, S, ts, strat):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, REPO=ROOT, S=str(S), TS=str(ts), STRAT=str(strat), MASTER_ADDR="127.0.0.1")
    port = _free_port()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", f"--master-port={port}", str(script)],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "RANK0OK" in r.stdout and "RANK1OK" in r.stdout


TABLE_WORKER = textwrap.dedent(r'''
    import os, sys
    sys.path.insert(0, os.environ["REPO"])
    import numpy as np, torch, torch.distributed as dist
    import oracle
    import importlib.util
    spec = importlib.util.spec_from_file_location("sharded", os.path.join(os.environ["REPO"], "paper_2203_14883_b200", "sharded.py"))
    sh = importlib.util.module_from_spec(spec); spec.loader.exec_module(sh)

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    K = int(os.environ["K"])
    V, w = 300, 5
    rng = np.random.default_rng(7)                      # same full state on every rank
    full = rng.standard_normal((V * K, w)).astype(np.float32)
    pos0 = rng.integers(0, K, V).astype(np.int32)
    splits = torch.tensor([0, 131, V], dtype=torch.int64)
    lo, hi = int(splits[rank]), int(splits[rank + 1])

    class CpuTableOps:                                  # test double: numpy + the oracle's state write
        def bucket(self, ids, splits, world):
            owner = np.searchsorted(splits.numpy()[1:-1], ids.numpy(), side="right")
            perm = np.argsort(owner, kind="stable").astype(np.int32)
            return torch.from_numpy(perm), torch.from_numpy(np.bincount(owner, minlength=world).astype(np.int64))
        def pack(self, perm, tensors):
            return [t[perm.long()].contiguous() for t in tensors]
        def invert(self, perm):
            inv = np.empty(len(perm), np.int32); inv[perm.numpy()] = np.arange(len(perm), dtype=np.int32)
            return torch.from_numpy(inv)
        def local_gather(self, ids, table, lo, n_global):
            return table[(ids - lo).long()].contiguous()
        def local_state_write(self, ids, ts, pairs, lo, n_global, K, pos, ts_table):
            loc = (ids.numpy() - lo).astype(np.int32)
            oracle.state_write(loc, ts.numpy(), n_nodes=hi - lo, K=K,
                               tables=[(r.numpy(), t.numpy()) for r, t in pairs],
                               pos=None if pos is None else pos.numpy())

    table = torch.from_numpy(full[lo * K:hi * K].copy())
    pos = torch.from_numpy(pos0[lo:hi].copy())
    tabs = sh.ShardedNodeTables(splits, sh.DistExchange(), CpuTableOps(), [table], K=K, pos=pos if K > 1 else None)
    q = np.random.default_rng(100 + rank).integers(0, V, 50).astype(np.int32)
    got = tabs.gather(torch.from_numpy(q))[0].numpy()
    assert np.array_equal(got, full.reshape(V, K * w)[q])
    evs = []
    for r in range(world):
        g = np.random.default_rng(200 + r)
        n = 40 + 9 * r
        evs.append(((g.zipf(1.5, n) % V).astype(np.int32), np.arange(n, dtype=np.float32),
                    g.standard_normal((n, w)).astype(np.float32)))
    ids, ts, rows = evs[rank]
    tabs.state_write(torch.from_numpy(ids), torch.from_numpy(ts), [torch.from_numpy(rows)])
    ref, ref_pos = full.copy(), pos0.copy()
    oracle.state_write(np.concatenate([e[0] for e in evs]), np.concatenate([e[1] for e in evs]), n_nodes=V, K=K,
                       tables=[(np.concatenate([e[2] for e in evs]), ref)], pos=ref_pos if K > 1 else None)
    assert np.array_equal(table.numpy(), ref[lo * K:hi * K])
    if K > 1:
        assert np.array_equal(pos.numpy(), ref_pos[lo:hi])
    dist.barrier()
    dist.destroy_process_group()
    print(f"RANK{rank}OK", flush=True)
''')


@pytest.mark.parametrize("K", [1, 3])
def test_sharded_node_tables_protocol_gloo_world2(tmp_path, K):
    """ShardedNodeTables over a real 2-process gloo all-to-all: gather returns
    the full tables' rows; state_write equals one sequential write of both ranks' events."""
    script = tmp_path / "table_worker.py"
    script.write_text(TABLE_WORKER)
    env = dict(os.environ, REPO=ROOT, K=str(K), MASTER_ADDR="127.0.0.1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(script)],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "RANK0OK" in r.stdout and "RANK1OK" in r.stdout
