"""Node-sharded sampling: the PROTOCOL MODEL in Python over torch.distributed.

The product node-sharded path is behind the C ABI (include/tgl.h: tgl_tcsr_build_range,
tgl_shard_create, tgl_sample_sharded, tgl_shard_gather, tgl_shard_state_write; Python:
`ShardSampler`): NCCL send/recv groups inside the library, any number of layers.  This module keeps
the same exchange written against torch.distributed all-to-all (pluggable ops / exchange), which
runs with gloo on CPU (tests/test_sharded_gloo.py, world 2) -- the host-side model of the protocol
-- and `edge_balanced_splits`, shared by both.

Node-sharded sampling: the T-CSR split by node ranges over the ranks.

For graphs larger than one GPU's HBM the T-CSR is split into contiguous node ranges balanced by
edges; the node v is owned by shard r with splits[r] <= v < splits[r+1].  One sampling call:

  1. K8  tgl_shard_bucket     stable bucketing of the local roots by owner shard (perm, counts)
  2. K7  tgl_gather           pack the requests (node, t, root key) in bucket order
  3.     all-to-all-v         requests to their owners (NCCL through torch.distributed)
  4. K4  tgl_sample_keyed     each owner samples the roots it received, with the roots' GLOBAL keys
                              (R#7), so the bits equal the replicated mode's
  5.     all-to-all-v         replies: per-root counts + (nbr, eid, dt) edges, per snapshot block
  6. K8b tgl_shard_unpermute  back to the original root order: the exact replicated-mode blocks

Steps 1, 2, 4, 6 are the library's kernels; 3 and 5 are the collective (the path's real exchange
step).  The exchange object is pluggable: `DistExchange` (torch.distributed all_to_all_single:
NCCL on GPUs, gloo on CPU tests) or a test double.  `ops` is pluggable the same way so the
exchange protocol can be exercised on CPU with world_size 2 (tests/test_sharded_gloo.py); on a GPU
`CudaOps` calls only libtgl.so.  Single layer (the C5 configuration); the multi-layer node-sharded
sampler is the C-ABI one (`tgl_sample_sharded`).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch


def edge_balanced_splits(indptr: torch.Tensor, world: int) -> torch.Tensor:
    """splits[r] = first node whose list starts at or after r * E_s / world (int64 [world+1])."""
    V = indptr.numel() - 1
    E = int(indptr[-1].item())
    targets = torch.tensor([E * r // world for r in range(world + 1)], dtype=torch.int64, device=indptr.device)
    s = torch.searchsorted(indptr[:V].contiguous(), targets, right=False)
    s[0], s[-1] = 0, V
    return torch.cummax(s, 0).values


class DistExchange:
    """all-to-all-v over torch.distributed (NCCL or gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def splits(self, send_counts: torch.Tensor) -> torch.Tensor:
        """Exchange per-peer element counts (int64 [world]) -> counts to receive from each peer."""
        recv = torch.empty_like(send_counts)
        self.dist.all_to_all_single(recv, send_counts.contiguous(), group=self.group)
        return recv

    def exchange(self, t: torch.Tensor, send_splits: Sequence[int], recv_splits: Sequence[int]) -> torch.Tensor:
        out = torch.empty((int(sum(recv_splits)),) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        self.dist.all_to_all_single(out, t.contiguous(), list(map(int, recv_splits)), list(map(int, send_splits)),
                                    group=self.group)
        return out


class CudaOps:
    """The product ops: libtgl.so kernels only."""

    def __init__(self, shard, fanout: int, strategy, n_snapshots: int, snapshot_len: float, max_roots: int):
        from . import Sampler
        import paper_2203_14883_b200 as tgl
        self.tgl = tgl
        self.sampler = Sampler(shard, max(max_roots, 1), [fanout], strategy, n_snapshots, snapshot_len)

    def bucket(self, roots, splits, world):
        return self.tgl.shard_bucket(roots, splits, world)

    def pack(self, perm, roots, root_ts, keys):
        r, t, k = self.tgl.gather(perm, [roots, root_ts, keys])
        return r, t, k

    def sample(self, roots, root_ts, keys, seed):
        """-> per snapshot (counts int32 [n], nbr, eid, dt) over the received roots."""
        n = roots.numel()
        blocks = self.sampler.run(roots, root_ts, root_keys=keys, seed=seed, n_roots=n)
        out = []
        for b in blocks:
            nnz = int(b.nnz_dev.item())
            cnt = self.tgl.offsets_to_counts(b.offsets, n)
            out.append((cnt, b.nbr[:nnz], b.eid[:nnz], b.dt[:nnz], b.offsets[: n + 1]))
        return out

    def unpermute(self, perm, counts, nbr, eid, dt):
        return self.tgl.shard_unpermute(perm, counts, nbr, eid, dt)


@dataclass
class ShardedBlock:
    offsets: torch.Tensor
    nbr: torch.Tensor
    eid: torch.Tensor
    dt: torch.Tensor


class NodeShardedSampler:
    """One rank's view of the node-sharded sampler (1 layer, S snapshots)."""

    def __init__(self, splits: torch.Tensor, exchange, ops, n_snapshots: int, seed: int):
        self.splits = splits
        self.ex = exchange
        self.ops = ops
        self.S = int(n_snapshots)
        self.seed = int(seed)

    def run(self, roots: torch.Tensor, root_ts: torch.Tensor, root_key_base: int) -> List[ShardedBlock]:
        W = self.ex.world
        n = roots.numel()
        dev = roots.device
        keys = torch.arange(root_key_base, root_key_base + n, dtype=torch.int64, device=dev)
        perm, counts = self.ops.bucket(roots, self.splits, W)                 # K8
        send_roots = counts.to(torch.int64)
        recv_roots = self.ex.splits(send_roots)
        sr, rr = send_roots.tolist(), recv_roots.tolist()
        p_nodes, p_ts, p_keys = self.ops.pack(perm, roots, root_ts, keys)     # K7 (bucket order)
        q_nodes = self.ex.exchange(p_nodes, sr, rr)                          # requests -> owners
        q_ts = self.ex.exchange(p_ts, sr, rr)
        q_keys = self.ex.exchange(p_keys, sr, rr)
        local = self.ops.sample(q_nodes, q_ts, q_keys, self.seed)            # K4 on the local shard
        seg = [0]
        for c in rr:
            seg.append(seg[-1] + int(c))
        out = []
        for (cnt, nbr, eid, dt, off) in local:
            bounds = off[torch.tensor(seg, dtype=torch.int64, device=off.device)].tolist()
            send_edges = [bounds[p + 1] - bounds[p] for p in range(W)]
            recv_edges = self.ex.splits(torch.tensor(send_edges, dtype=torch.int64, device=dev)).tolist()
            r_cnt = self.ex.exchange(cnt, rr, sr)                            # replies -> sources
            r_nbr = self.ex.exchange(nbr, send_edges, recv_edges)
            r_eid = self.ex.exchange(eid, send_edges, recv_edges)
            r_dt = self.ex.exchange(dt, send_edges, recv_edges)
            o, nb, ed, d = self.ops.unpermute(perm, r_cnt, r_nbr, r_eid, r_dt)  # K8b
            out.append(ShardedBlock(o, nb, ed, d))
        return out


class CudaTableOps:
    """Product ops of the sharded node tables: libtgl.so kernels only."""

    def __init__(self):
        import paper_2203_14883_b200 as tgl
        self.tgl = tgl

    def bucket(self, ids, splits, world):
        return self.tgl.shard_bucket(ids, splits, world)

    def pack(self, perm, tensors):
        return self.tgl.gather(perm, tensors)

    def invert(self, perm):
        return self.tgl.perm_invert(perm)

    def local_gather(self, ids, table, lo, n_global):
        out = torch.empty((ids.numel(),) + tuple(table.shape[1:]), dtype=table.dtype, device=table.device)
        self.tgl.gather_rows_at(ids, table, lo, n_global, out)
        return out

    def local_state_write(self, ids, ts, pairs, lo, n_global, K, pos, ts_table):
        self.tgl.state_write_at(ids, ts, pairs, node_lo=lo, n_nodes_global=n_global, K=K, pos=pos, ts_table=ts_table)


class ShardedNodeTables:
    """Node memory / mailbox sharded by the node-sharded T-CSR's ranges (MAG's
    121 M x (100 + K x 428) fp32 state does not fit one GPU).  Rank r holds the rows of
    nodes [splits[r], splits[r+1]); each local table is [n_local * K, ...] (K ring slots per node,
    state-write layout; K = 1 for memory).

      gather(ids)             Fig. 2 step 2 across shards: owner bucketing (K8), all-to-all-v of the
                              ids, local tgl_gather, all-to-all-v of the rows back, request order
                              restored by tgl_gather through the inverse permutation.  Returns each
                              table's rows (a node's whole K-slot ring per id).
      state_write(ids, ts, rows)
                              Fig. 2 step 6 across shards: the events go to their owners (stable
                              bucketing: each owner receives them in (source rank, batch index)
                              order -- the global event order, R#25) and are applied there by
                              tgl_state_write.
    """

    def __init__(self, splits: torch.Tensor, exchange, ops, tables: Sequence[torch.Tensor], K: int = 1,
                 pos: Optional[torch.Tensor] = None, ts_table: Optional[torch.Tensor] = None):
        self.splits = splits
        self.ex = exchange
        self.ops = ops
        self.tables = list(tables)
        self.K = int(K)
        self.pos = pos
        self.ts_table = ts_table
        r = exchange.rank
        self.lo, self.hi = int(splits[r]), int(splits[r + 1])
        self.n_global = int(splits[-1])

    def _route(self, ids):
        W = self.ex.world
        perm, counts = self.ops.bucket(ids, self.splits, W)
        send = counts.to(torch.int64)
        recv = self.ex.splits(send)
        return perm, send.tolist(), recv.tolist()

    def gather(self, ids: torch.Tensor) -> List[torch.Tensor]:
        perm, sr, rr = self._route(ids)
        q_ids = self.ex.exchange(self.ops.pack(perm, [ids])[0], sr, rr)
        inv = self.ops.invert(perm)
        outs = []
        for t in self.tables:
            node_rows = t.reshape((t.shape[0] // self.K, -1) if t.dim() > 1 or self.K > 1 else (t.shape[0],))
            rows = self.ops.local_gather(q_ids, node_rows, self.lo, self.n_global)
            back = self.ex.exchange(rows, rr, sr)
            outs.append(self.ops.pack(inv, [back])[0])
        return outs

    def state_write(self, ids: torch.Tensor, ts: torch.Tensor, rows: Sequence[torch.Tensor]) -> None:
        perm, sr, rr = self._route(ids)
        packed = self.ops.pack(perm, [ids, ts] + list(rows))
        recv = [self.ex.exchange(x, sr, rr) for x in packed]
        q_ids, q_ts, q_rows = recv[0], recv[1], recv[2:]
        self.ops.local_state_write(q_ids, q_ts, list(zip(q_rows, self.tables)), self.lo, self.n_global, self.K,
                                   self.pos, self.ts_table)


def slice_shard(g, lo: int, hi: int):
    """Setup helper: the shard of a full T-CSR for nodes [lo, hi) as its own handle (copies)."""
    import paper_2203_14883_b200 as tgl
    a, b = int(g.indptr[lo].item()), int(g.indptr[hi].item())
    indptr = (g.indptr[lo:hi + 1] - a).contiguous()
    sh = tgl.wrap(indptr, g.nbr[a:b].clone(), g.ts[a:b].clone(), g.eid[a:b].clone())
    tgl.set_node_base(sh, lo)
    return sh
