"""TGL hot path on B200 (arXiv 2203.14883): T-CSR build, parallel temporal sampler, gather.

Thin Python binding over ``libtgl.so`` (C ABI: ``include/tgl.h``).  PyTorch provides device
memory and the current CUDA stream; every step of the path runs in the library's sm_100a
kernels.  There is no CPU fallback: importing this package without the built library raises,
and every call requires CUDA tensors.

    g = build(src, dst, ts, eid=None, n_nodes=V, add_reverse=True)
    blocks = sample(g, roots, root_ts, fanouts=[10], strategy="most_recent",  # Alg. 1
                    n_snapshots=1, snapshot_len=float("inf"), seed=0, root_key_base=0)
    outs = gather(ids, [memory, mailbox, ...], n_ids_dev=None)                 # Fig. 2 step 2
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import MOST_RECENT, UNIFORM, TGLError

_L = _lib.load()

__all__ = ["TCSR", "Block", "Sampler", "build", "wrap", "aux_bytes", "sample", "gather", "check", "shard_bucket",
           "set_node_base", "shard_unpermute", "offsets_to_counts", "block_digest", "tcsr_indptr", "build_range", "batch_roots",
           "nccl_id", "ShardGroup", "ShardSampler",
           "MOST_RECENT", "UNIFORM", "TGLError", "lib_path"]

lib_path = _lib.LIB_PATH


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _rc(code: int, what: str):
    if code != _lib.OK:
        raise TGLError(code, what, _L)


def _cuda(t: torch.Tensor, dtype: torch.dtype, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    return t.contiguous()


def _strategy(s) -> int:
    if isinstance(s, str):
        return {"most_recent": MOST_RECENT, "uniform": UNIFORM}[s]
    return int(s)


class TCSR:
    """A built T-CSR: indptr int64 [V+1]; nbr int32, ts float32, eid int32 [E_s] (+ sampler aux buffer)."""

    def __init__(self, indptr, nbr, ts, eid, n_nodes, handle, index=None, ts_storage=None):
        self.indptr, self.nbr, self.ts, self.eid = indptr, nbr, ts, eid
        self.index = index
        self._ts_storage = ts_storage
        self.n_nodes = int(n_nodes)
        self.n_stored = int(nbr.numel())
        self.node_lo = 0
        self._h = handle

    @property
    def handle(self):
        return self._h

    @property
    def codec(self) -> dict:
        """tgl_tcsr_codec: {"n_codes": distinct times coded (0 = no time codec), "packed": 8-byte slot
        records -- 0 no, 1 with time codes, 2 with integer times (< 2^24, without time codes)}."""
        n, pk = ctypes.c_int32(), ctypes.c_int32()
        _rc(_L.tgl_tcsr_codec(self._h, ctypes.byref(n), ctypes.byref(pk)), "tgl_tcsr_codec")
        return {"n_codes": n.value, "packed": pk.value}

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _L is not None:
            _L.tgl_tcsr_destroy(h)


def build_workspace_bytes(n_edges: int, n_nodes: int, add_reverse: bool) -> int:
    b = ctypes.c_size_t()
    _rc(_L.tgl_tcsr_build_workspace(int(n_edges), int(n_nodes), int(add_reverse), ctypes.byref(b)),
        "tgl_tcsr_build_workspace")
    return b.value


def aux_bytes(n_stored: int, n_nodes: int) -> int:
    b = ctypes.c_size_t()
    _rc(_L.tgl_tcsr_aux_bytes(int(n_stored), int(n_nodes), ctypes.byref(b)), "tgl_tcsr_aux_bytes")
    return b.value


def _ts_buffer(n: int, dev) -> (torch.Tensor, torch.Tensor):
    """float32 [n] view of a 64-byte aligned buffer padded to a multiple of 16 floats (the sampler
    reads timestamps in aligned 64-byte groups)."""
    storage = torch.empty(max((n + 15) // 16 * 16, 16), dtype=torch.float32, device=dev)
    assert storage.data_ptr() % 64 == 0
    return storage[:n], storage


def build(src: torch.Tensor, dst: torch.Tensor, ts: torch.Tensor, eid: Optional[torch.Tensor] = None, *,
          n_nodes: int, add_reverse: bool, workspace: Optional[torch.Tensor] = None, with_index: bool = True,
          stream=None) -> TCSR:
    """tgl_tcsr_build: T-CSR of a chronological stream + the sampler aux buffer."""
    src = _cuda(src, torch.int32, "src")
    dst = _cuda(dst, torch.int32, "dst")
    ts = _cuda(ts, torch.float32, "ts")
    if eid is not None:
        eid = _cuda(eid, torch.int32, "eid")
    E = src.numel()
    Es = E * (2 if add_reverse else 1)
    dev = src.device
    indptr = torch.empty(n_nodes + 1, dtype=torch.int64, device=dev)
    nbr = torch.empty(Es, dtype=torch.int32, device=dev)
    ts_out, ts_storage = _ts_buffer(Es, dev)
    eid_out = torch.empty(Es, dtype=torch.int32, device=dev)
    ib = aux_bytes(Es, n_nodes) if with_index else 0
    index = torch.empty(ib, dtype=torch.uint8, device=dev) if with_index else None
    wsb = build_workspace_bytes(E, n_nodes, add_reverse)
    if workspace is None or workspace.numel() < wsb:
        workspace = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    h = ctypes.c_void_p()
    _rc(_L.tgl_tcsr_build(_ptr(src), _ptr(dst), _ptr(ts), _ptr(eid), E, int(n_nodes), int(add_reverse),
                          _ptr(indptr), _ptr(nbr), _ptr(ts_storage), _ptr(eid_out), _ptr(index), ib,
                          _ptr(workspace), wsb, _stream(stream), ctypes.byref(h)), "tgl_tcsr_build")
    return TCSR(indptr, nbr, ts_out, eid_out, n_nodes, h, index, ts_storage)


def wrap(indptr: torch.Tensor, nbr: torch.Tensor, ts: torch.Tensor, eid: torch.Tensor, *,
         with_index: bool = True, stream=None) -> TCSR:
    """tgl_tcsr_wrap: handle over existing T-CSR arrays (e.g. broadcast from another rank)."""
    indptr = _cuda(indptr, torch.int64, "indptr")
    nbr = _cuda(nbr, torch.int32, "nbr")
    eid = _cuda(eid, torch.int32, "eid")
    n = nbr.numel()
    ts_view, ts_storage = _ts_buffer(n, nbr.device)
    ts_view.copy_(_cuda(ts, torch.float32, "ts"))
    V = indptr.numel() - 1
    ib = aux_bytes(n, V) if with_index else 0
    index = torch.empty(ib, dtype=torch.uint8, device=nbr.device) if with_index else None
    if with_index:
        _rc(_L.tgl_tcsr_aux_build(_ptr(indptr), _ptr(ts_storage), _ptr(nbr), _ptr(eid), V, n, _ptr(index), ib,
                                  _stream(stream)), "tgl_tcsr_aux_build")
    h = ctypes.c_void_p()
    _rc(_L.tgl_tcsr_wrap(_ptr(indptr), _ptr(nbr), _ptr(ts_storage), _ptr(eid), _ptr(index), ib,
                         indptr.numel() - 1, n, ctypes.byref(h)), "tgl_tcsr_wrap")
    return TCSR(indptr, nbr, ts_view, eid, indptr.numel() - 1, h, index, ts_storage)


@dataclass
class Block:
    """One (layer, snapshot) message-flow block at capacity size; n_roots / nnz live on the device."""
    offsets: torch.Tensor
    nbr: torch.Tensor
    eid: torch.Tensor
    dt: torch.Tensor
    ts_edge: Optional[torch.Tensor]
    n_roots_dev: torch.Tensor
    nnz_dev: torch.Tensor
    # dedup (R#27): distinct (node, hop time) pairs of the outputs, first appearance order
    src_index: Optional[torch.Tensor] = None
    uniq_node: Optional[torch.Tensor] = None
    uniq_ts: Optional[torch.Tensor] = None
    n_uniq_dev: Optional[torch.Tensor] = None

    def batch(self, r0: int, r1: int):
        """Views of roots [r0, r1) of this block -- e.g. one mini-batch of a many-batch (epoch-mode)
        call: (offsets rebased to the batch, nbr, eid, dt[, ts_edge]).  Host-synchronising (reads
        two offsets); no copies of the edge arrays."""
        o = self.offsets[r0:r1 + 1]
        e0, e1 = int(o[0].item()), int(o[-1].item())
        te = None if self.ts_edge is None else self.ts_edge[e0:e1]
        return o - e0, self.nbr[e0:e1], self.eid[e0:e1], self.dt[e0:e1], te

    def trimmed(self):
        """Host-synchronising view: (offsets[:n+1], nbr[:nnz], eid[:nnz], dt[:nnz], ts_edge[:nnz])."""
        n, nnz = int(self.n_roots_dev.item()), int(self.nnz_dev.item())
        te = None if self.ts_edge is None else self.ts_edge[:nnz]
        return self.offsets[: n + 1], self.nbr[:nnz], self.eid[:nnz], self.dt[:nnz], te


def _alloc_blocks(dev, rc_, ec_, L: int, S: int, want_ts_edge_last: bool = False) -> List["Block"]:
    """Device blocks (l, s) at index l*S + s with the capacities of tgl_sample_capacity."""
    scal = torch.zeros(2 * L * S, dtype=torch.int64, device=dev)
    blocks = []
    for l in range(L):
        for s in range(S):
            need_ts = l < L - 1 or want_ts_edge_last
            j = l * S + s
            blocks.append(Block(
                offsets=torch.empty(rc_[l] + 1, dtype=torch.int64, device=dev),
                nbr=torch.empty(ec_[l], dtype=torch.int32, device=dev),
                eid=torch.empty(ec_[l], dtype=torch.int32, device=dev),
                dt=torch.empty(ec_[l], dtype=torch.float32, device=dev),
                ts_edge=torch.empty(ec_[l], dtype=torch.float32, device=dev) if need_ts else None,
                n_roots_dev=scal[2 * j: 2 * j + 1], nnz_dev=scal[2 * j + 1: 2 * j + 2]))
    return blocks


def _c_blocks(blocks, rc_, ec_, S: int):
    arr = (_lib.Block * len(blocks))()
    for j, b in enumerate(blocks):
        l = j // S
        arr[j] = _lib.Block(rc_[l], ec_[l], b.offsets.data_ptr(), b.nbr.data_ptr(), b.eid.data_ptr(),
                            b.dt.data_ptr(), 0 if b.ts_edge is None else b.ts_edge.data_ptr(),
                            b.n_roots_dev.data_ptr(), b.nnz_dev.data_ptr())
    return arr


class Sampler:
    """Preallocated outputs + workspace for repeated tgl_sample calls of up to max_roots roots."""

    def __init__(self, g: TCSR, max_roots: int, fanouts: Sequence[int], strategy="most_recent",
                 n_snapshots: int = 1, snapshot_len: float = math.inf, device=None, want_ts_edge_last=False,
                 hop_time: str = "edge", replacement: bool = False, dedup: bool = False,
                 edge_valid: Optional[torch.Tensor] = None, fused_gather=None):
        """hop_time: "edge" (R#4) or "root" (R#23, hop roots carry the root time); replacement:
        uniform with replacement (R#24); dedup: per-block distinct (node, hop time) lists feeding
        the next layer (R#27); edge_valid: int32/uint32 CUDA bitmask over edge ids (R#28), invalid
        edges are not candidates -- its contents may change between runs (tgl_edge_valid_set).
        All map to tgl_sample_ex's options."""
        self.g = g
        if hop_time not in ("edge", "root"):
            raise ValueError("hop_time must be 'edge' or 'root'")
        self._opts = _lib.SampleOptions(1 if hop_time == "root" else 0, 1 if replacement else 0, 1 if dedup else 0)
        self.edge_valid = edge_valid
        if edge_valid is not None:
            if not (edge_valid.is_cuda and edge_valid.dtype in (torch.int32, torch.uint32) and edge_valid.is_contiguous()):
                raise TypeError("edge_valid must be a contiguous CUDA int32/uint32 bitmask")
            self._opts.edge_valid = edge_valid.data_ptr()
        self.fused_outs = []
        if fused_gather:
            # tgl_fused_gather: [(table, "node" | "edge")] -> rows of the last layer's outputs, written by the
            # copy kernel into self.fused_outs[j] ([edges_cap, ...], row i = output i of the last block)
            if len(fused_gather) > _lib.MAX_FUSED_GATHER:
                raise ValueError("too many fused gather tables")
            self._fg = _lib.FusedGather()
            self._fg.n_tables = len(fused_gather)
            self._fused_spec = list(fused_gather)
            self._opts.gather = ctypes.pointer(self._fg)
        self._default_opts = hop_time == "edge" and not replacement and not dedup and edge_valid is None \
            and not fused_gather
        self.dedup = bool(dedup)
        if dedup and hop_time == "edge":
            want_ts_edge_last = True
        self.fanouts = [int(k) for k in fanouts]
        self.L, self.S = len(self.fanouts), int(n_snapshots)
        self.strategy = _strategy(strategy)
        self.snapshot_len = float(snapshot_len)
        self.max_roots = int(max_roots)
        dev = g.nbr.device if device is None else device
        rc_, ec_, wsb = self.capacity(self.max_roots)
        self.roots_cap, self.edges_cap = rc_, ec_
        self.workspace = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        self.ws_bytes = wsb
        self.blocks: List[Block] = _alloc_blocks(dev, rc_, ec_, self.L, self.S, want_ts_edge_last)
        self._c_dedup = None
        if dedup:
            uscal = torch.zeros(self.L * self.S, dtype=torch.int64, device=dev)
            self._c_dedup = (_lib.DedupBlock * len(self.blocks))()
            for j, b in enumerate(self.blocks):
                l = j // self.S
                b.src_index = torch.empty(ec_[l], dtype=torch.int32, device=dev)
                b.uniq_node = torch.empty(ec_[l], dtype=torch.int32, device=dev)
                b.uniq_ts = torch.empty(ec_[l], dtype=torch.float32, device=dev)
                b.n_uniq_dev = uscal[j:j + 1]
                self._c_dedup[j] = _lib.DedupBlock(ec_[l], b.src_index.data_ptr(), b.uniq_node.data_ptr(),
                                                   b.uniq_ts.data_ptr(), b.n_uniq_dev.data_ptr())
        self._c_blocks = _c_blocks(self.blocks, rc_, ec_, self.S)
        if fused_gather:
            for j, (t, by) in enumerate(self._fused_spec):
                if by not in ("node", "edge") or not (t.is_cuda and t.is_contiguous()):
                    raise ValueError("fused gather: (contiguous CUDA table, 'node' | 'edge')")
                rb = t.element_size() * int(np.prod(t.shape[1:], dtype=np.int64))
                o = torch.empty((ec_[-1],) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
                self.fused_outs.append(o)
                self._fg.tables[j] = _lib.FusedTable(t.data_ptr(), t.shape[0], rb, o.data_ptr(), 1 if by == "edge" else 0)
        self._fan = (ctypes.c_int32 * self.L)(*self.fanouts)

    def capacity(self, n_roots: int):
        rc_ = (ctypes.c_int64 * self.L)()
        ec_ = (ctypes.c_int64 * self.L)()
        wsb = ctypes.c_size_t()
        fan = (ctypes.c_int32 * self.L)(*self.fanouts)
        _rc(_L.tgl_sample_capacity_ex(int(n_roots), self.L, fan, self.S, self.strategy, self.snapshot_len,
                                      ctypes.byref(self._opts), rc_, ec_, ctypes.byref(wsb)), "tgl_sample_capacity_ex")
        return list(rc_), list(ec_), wsb.value

    def run(self, roots: torch.Tensor, root_ts: torch.Tensor, *, seed: int = 0, root_key_base: int = 0,
            root_keys: Optional[torch.Tensor] = None, n_roots: Optional[int] = None, stream=None) -> List[Block]:
        """tgl_sample (or tgl_sample_keyed when root_keys, int64 bit patterns of uint64 keys, is given)
        on the current (or given) stream; no host synchronisation."""
        n = roots.numel() if n_roots is None else int(n_roots)
        if n < 0 or n > self.max_roots:
            raise ValueError(f"{n} roots outside [0, max_roots {self.max_roots}]")
        if not (roots.is_cuda and roots.dtype == torch.int32 and root_ts.is_cuda and root_ts.dtype == torch.float32):
            raise TypeError("roots must be CUDA int32 and root_ts CUDA float32 (no CPU fallback)")
        # raw data pointers go to the library: the tensors must be dense and hold n elements
        if not (roots.is_contiguous() and root_ts.is_contiguous()):
            raise ValueError("roots and root_ts must be contiguous")
        if n > roots.numel() or n > root_ts.numel():
            raise ValueError(f"n_roots {n} exceeds roots ({roots.numel()}) or root_ts ({root_ts.numel()})")
        if root_keys is not None:
            if not (root_keys.is_cuda and root_keys.dtype == torch.int64):
                raise TypeError("root_keys must be a CUDA int64 tensor (uint64 bit patterns)")
            if not root_keys.is_contiguous() or n > root_keys.numel():
                raise ValueError("root_keys must be contiguous with at least n_roots elements")
            _rc(_L.tgl_sample_ex(self.g.handle, _ptr(roots), _ptr(root_ts), _ptr(root_keys), n, self.L, self._fan,
                                 self.strategy, self.S, self.snapshot_len, int(seed) & 0xFFFFFFFFFFFFFFFF, 0,
                                 ctypes.byref(self._opts), self._c_blocks, self._c_dedup, _ptr(self.workspace),
                                 self.ws_bytes, _stream(stream)), "tgl_sample_ex")
            return self.blocks
        if self._default_opts:
            _rc(_L.tgl_sample(self.g.handle, _ptr(roots), _ptr(root_ts), n, self.L, self._fan, self.strategy, self.S,
                              self.snapshot_len, int(seed) & 0xFFFFFFFFFFFFFFFF, int(root_key_base) & 0xFFFFFFFFFFFFFFFF,
                              self._c_blocks, _ptr(self.workspace), self.ws_bytes, _stream(stream)), "tgl_sample")
        else:
            _rc(_L.tgl_sample_ex(self.g.handle, _ptr(roots), _ptr(root_ts), None, n, self.L, self._fan, self.strategy,
                                 self.S, self.snapshot_len, int(seed) & 0xFFFFFFFFFFFFFFFF,
                                 int(root_key_base) & 0xFFFFFFFFFFFFFFFF, ctypes.byref(self._opts), self._c_blocks,
                                 self._c_dedup, _ptr(self.workspace), self.ws_bytes, _stream(stream)), "tgl_sample_ex")
        return self.blocks


def sample(g: TCSR, roots: torch.Tensor, root_ts: torch.Tensor, *, fanouts: Sequence[int],
           strategy="most_recent", n_snapshots: int = 1, snapshot_len: float = math.inf, seed: int = 0,
           root_key_base: int = 0, stream=None, hop_time: str = "edge", replacement: bool = False,
           dedup: bool = False, edge_valid: Optional[torch.Tensor] = None) -> List[Block]:
    """tgl_sample (Alg. 1): returns L*S blocks, block (l, s) at index l*S + s.  hop_time /
    replacement select the variants of tgl_sample_ex (R#23, R#24)."""
    roots = _cuda(roots, torch.int32, "roots")
    root_ts = _cuda(root_ts, torch.float32, "root_ts")
    s = Sampler(g, max(roots.numel(), 1), fanouts, strategy, n_snapshots, snapshot_len, hop_time=hop_time,
                replacement=replacement, dedup=dedup, edge_valid=edge_valid)
    return s.run(roots, root_ts, seed=seed, root_key_base=root_key_base, n_roots=roots.numel(), stream=stream)


def gather(ids: torch.Tensor, tables: Sequence[torch.Tensor], *, n_ids_dev: Optional[torch.Tensor] = None,
           outs: Optional[Sequence[torch.Tensor]] = None, stream=None) -> List[torch.Tensor]:
    """tgl_gather: out_t[i] = table_t[ids[i]] (rows of any width); id -1 -> zero row."""
    ids = _cuda(ids, torch.int32, "ids")
    n = ids.numel()
    if len(tables) > _lib.MAX_GATHER_TABLES:
        raise ValueError("too many tables")
    res, arr = [], (_lib.GatherTable * max(len(tables), 1))()
    for j, t in enumerate(tables):
        if not t.is_cuda or not t.is_contiguous():
            raise TypeError("gather tables must be contiguous CUDA tensors")
        rows = t.shape[0]
        row_bytes = t.element_size() * (t[0].numel() if t.dim() > 1 else 1)
        o = outs[j] if outs is not None else torch.empty((n,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        res.append(o)
        arr[j] = _lib.GatherTable(t.data_ptr(), rows, row_bytes, o.data_ptr())
    _rc(_L.tgl_gather(_ptr(ids), n, _ptr(n_ids_dev), arr, len(tables), _stream(stream)), "tgl_gather")
    return res


class StateWriter:
    """tgl_state_write (Fig. 2 step 6, R#25) with a preallocated workspace for up to max_events
    events: node memory / mailbox rings updated in place, events applied in batch order."""

    def __init__(self, n_nodes: int, max_events: int, device=None):
        self.n_nodes = int(n_nodes)
        self.max_events = int(max_events)
        b = ctypes.c_size_t()
        _rc(_L.tgl_state_write_workspace(self.max_events, self.n_nodes, ctypes.byref(b)), "tgl_state_write_workspace")
        self.ws_bytes = b.value
        self.workspace = torch.empty(max(b.value, 1), dtype=torch.uint8, device=device or "cuda")

    def __call__(self, ids: torch.Tensor, ts: Optional[torch.Tensor], tables, *, K: int = 1,
                 pos: Optional[torch.Tensor] = None, ts_table: Optional[torch.Tensor] = None, stream=None):
        """tables: [(rows [n, ...], table [n_nodes * K, ...])]; pos: int32 [n_nodes] ring cursors
        (required for K > 1); ts_table: float32 [n_nodes * K] (optional)."""
        ids = _cuda(ids, torch.int32, "ids")
        n = ids.numel()
        if n > self.max_events:
            raise ValueError(f"{n} events > max_events {self.max_events}")
        if ts is not None:
            ts = _cuda(ts, torch.float32, "ts")
        arr = (_lib.StateTable * max(len(tables), 1))()
        for j, (rows, table) in enumerate(tables):
            if not (rows.is_cuda and table.is_cuda and rows.is_contiguous() and table.is_contiguous()):
                raise TypeError("state rows / tables must be contiguous CUDA tensors")
            rb = rows.element_size() * (rows[0].numel() if rows.dim() > 1 else 1) if rows.shape[0] else \
                rows.element_size() * int(np.prod(rows.shape[1:], dtype=np.int64))
            if table.numel() * table.element_size() != self.n_nodes * K * rb:
                raise ValueError("table must hold n_nodes * K rows of the rows' width")
            arr[j] = _lib.StateTable(rows.data_ptr(), rb, table.data_ptr())
        if pos is not None:
            pos = _cuda(pos, torch.int32, "pos")
        if ts_table is not None:
            ts_table = _cuda(ts_table, torch.float32, "ts_table")
        _rc(_L.tgl_state_write(_ptr(ids), _ptr(ts), n, self.n_nodes, int(K), _ptr(pos), _ptr(ts_table), arr,
                               len(tables), _ptr(self.workspace), self.ws_bytes, _stream(stream)), "tgl_state_write")


def state_write(ids, ts, tables, *, n_nodes: int, K: int = 1, pos=None, ts_table=None, stream=None):
    """One-shot tgl_state_write (allocates its workspace)."""
    StateWriter(n_nodes, max(ids.numel(), 1), device=ids.device)(ids, ts, tables, K=K, pos=pos, ts_table=ts_table,
                                                                 stream=stream)


def chunk_schedule(n_edges: int, batch_size: int, chunk_size: int, epoch: int, seed: int, device="cuda",
                   stream=None):
    """tgl_chunk_schedule (Alg. 2, R#26): (first_edge int64 [cap] device, n_batches int64 [1] device)
    -- the first nb entries are the epoch's batch starts (no host sync)."""
    cap = max(int(n_edges) // int(batch_size), 1)
    first = torch.empty(cap, dtype=torch.int64, device=device)
    nb = torch.empty(1, dtype=torch.int64, device=device)
    _rc(_L.tgl_chunk_schedule(int(n_edges), int(batch_size), int(chunk_size), int(epoch), int(seed) & 0xFFFFFFFFFFFFFFFF,
                              _ptr(first), cap, _ptr(nb), _stream(stream)), "tgl_chunk_schedule")
    return first, nb


def edge_valid_set(valid: torch.Tensor, eids: torch.Tensor, value: bool, n_bits: Optional[int] = None,
                   stream=None) -> None:
    """tgl_edge_valid_set (R#28): set (True) / clear (False) the bits of eids in the bitmask."""
    eids = _cuda(eids, torch.int32, "eids")
    nb = valid.numel() * 32 if n_bits is None else int(n_bits)
    _rc(_L.tgl_edge_valid_set(_ptr(valid), nb, _ptr(eids), eids.numel(), 1 if value else 0, _stream(stream)),
        "tgl_edge_valid_set")


def perm_invert(perm: torch.Tensor, stream=None) -> torch.Tensor:
    """tgl_perm_invert: inv[perm[j]] = j (int32)."""
    perm = _cuda(perm, torch.int32, "perm")
    inv = torch.empty_like(perm)
    _rc(_L.tgl_perm_invert(_ptr(perm), perm.numel(), _ptr(inv), _stream(stream)), "tgl_perm_invert")
    return inv


def gather_rows_at(ids: torch.Tensor, table: torch.Tensor, row_lo: int, n_rows_global: int, out: torch.Tensor,
                   n_ids_dev: Optional[torch.Tensor] = None, stream=None) -> None:
    """tgl_gather on a shard-local table holding global rows [row_lo, row_lo + table.shape[0]),
    addressed with GLOBAL ids: the table base is offset by -row_lo rows (the ids a shard receives
    are >= row_lo by construction of the owner bucketing); ids >= n_rows_global give zero rows."""
    ids = _cuda(ids, torch.int32, "ids")
    rb = table.element_size() * (table[0].numel() if table.dim() > 1 else 1) if table.shape[0] else \
        table.element_size() * int(np.prod(table.shape[1:], dtype=np.int64))
    arr = (_lib.GatherTable * 1)()
    arr[0] = _lib.GatherTable(table.data_ptr() - int(row_lo) * rb, int(n_rows_global), rb, out.data_ptr())
    _rc(_L.tgl_gather(_ptr(ids), ids.numel(), _ptr(n_ids_dev), arr, 1, _stream(stream)), "tgl_gather")


def state_write_at(ids: torch.Tensor, ts: Optional[torch.Tensor], tables, *, node_lo: int, n_nodes_global: int,
                   K: int = 1, pos: Optional[torch.Tensor] = None, ts_table: Optional[torch.Tensor] = None,
                   stream=None) -> None:
    """tgl_state_write on shard-local state holding the rings of global nodes [node_lo, ...) and
    addressed with GLOBAL ids (base pointers offset by -node_lo nodes; the owner bucketing only
    sends a shard ids >= node_lo).  tables: [(rows [n, ...], local table [n_local * K, ...])]."""
    ids = _cuda(ids, torch.int32, "ids")
    n = ids.numel()
    lo = int(node_lo)
    arr = (_lib.StateTable * max(len(tables), 1))()
    for j, (rows, table) in enumerate(tables):
        rb = table.element_size() * (table[0].numel() if table.dim() > 1 else 1) if table.shape[0] else \
            table.element_size() * int(np.prod(table.shape[1:], dtype=np.int64))
        arr[j] = _lib.StateTable(rows.data_ptr() if n else None, rb, table.data_ptr() - lo * K * rb)
    b = ctypes.c_size_t()
    _rc(_L.tgl_state_write_workspace(n, int(n_nodes_global), ctypes.byref(b)), "tgl_state_write_workspace")
    ws = torch.empty(max(b.value, 1), dtype=torch.uint8, device=ids.device)
    pos_p = None if pos is None else pos.data_ptr() - lo * 4
    tst_p = None if ts_table is None else ts_table.data_ptr() - lo * K * 4
    _rc(_L.tgl_state_write(_ptr(ids), _ptr(ts), n, int(n_nodes_global), int(K), pos_p, tst_p, arr, len(tables),
                           _ptr(ws), b.value, _stream(stream)), "tgl_state_write")


def block_digest(block: Block, bounds: torch.Tensor, stream=None) -> torch.Tensor:
    """tgl_block_digest: per-batch FNV-1a-64 of a block (int64 tensor holding the uint64 bit
    patterns); batch j = the block's roots [bounds[j], bounds[j+1])."""
    bounds = _cuda(bounds, torch.int64, "bounds")
    nb = max(bounds.numel() - 1, 0)
    out = torch.empty(nb, dtype=torch.int64, device=bounds.device)
    _rc(_L.tgl_block_digest(_ptr(block.offsets), _ptr(block.nbr), _ptr(block.eid), _ptr(block.dt), _ptr(bounds), nb,
                            _ptr(out), _stream(stream)), "tgl_block_digest")
    return out


def batch_roots(src: torch.Tensor, dst: torch.Tensor, neg: torch.Tensor, ts: torch.Tensor, first_root: int,
                n_roots: int, out: Optional[tuple] = None, stream=None):
    """tgl_batch_roots: roots [first_root, first_root + n_roots) of a mini-batch of positive edges +
    negatives (R#16: src_i, dst_i, neg_i at ts_i); the arrays start at edge first_root // 3."""
    src = _cuda(src, torch.int32, "src")
    dst = _cuda(dst, torch.int32, "dst")
    neg = _cuda(neg, torch.int32, "neg")
    ts = _cuda(ts, torch.float32, "ts")
    n = int(n_roots)
    need = (int(first_root) + n - 1) // 3 + 1 - int(first_root) // 3 if n else 0
    if min(src.numel(), dst.numel(), neg.numel(), ts.numel()) < need:
        raise ValueError(f"the edge arrays must hold {need} edges")
    r, t = out if out is not None else (torch.empty(n, dtype=torch.int32, device=src.device),
                                        torch.empty(n, dtype=torch.float32, device=src.device))
    _rc(_L.tgl_batch_roots(_ptr(src), _ptr(dst), _ptr(neg), _ptr(ts), int(first_root), n, _ptr(r), _ptr(t),
                           _stream(stream)), "tgl_batch_roots")
    return r, t


def check(g: Optional[TCSR] = None, stream=None) -> int:
    """tgl_check: synchronise and return (and clear) the sticky device error code (0 = none)."""
    return _L.tgl_check(None if g is None else g.handle, _stream(stream))


def set_node_base(g: TCSR, node_lo: int) -> None:
    """tgl_tcsr_set_node_base: g holds the lists of global nodes [node_lo, node_lo + g.n_nodes)."""
    _rc(_L.tgl_tcsr_set_node_base(g.handle, int(node_lo)), "tgl_tcsr_set_node_base")
    g.node_lo = int(node_lo)


def offsets_to_counts(offsets: torch.Tensor, n: int, out: Optional[torch.Tensor] = None, stream=None):
    """tgl_offsets_to_counts: per-root counts (int32) of a CSR block."""
    offsets = _cuda(offsets, torch.int64, "offsets")
    out = torch.empty(max(n, 0), dtype=torch.int32, device=offsets.device) if out is None else out
    _rc(_L.tgl_offsets_to_counts(_ptr(offsets), int(n), _ptr(out), _stream(stream)), "tgl_offsets_to_counts")
    return out


def shard_unpermute(perm: torch.Tensor, counts_in: torch.Tensor, nbr_in: torch.Tensor, eid_in: torch.Tensor,
                    dt_in: torch.Tensor, stream=None):
    """tgl_shard_unpermute: CSR block in bucket order (per-root counts) -> the same block in original
    root order (offsets, nbr, eid, dt)."""
    perm = _cuda(perm, torch.int32, "perm")
    counts_in = _cuda(counts_in, torch.int32, "counts_in")
    n = perm.numel()
    dev = perm.device
    wsb = ctypes.c_size_t()
    _rc(_L.tgl_shard_unpermute_workspace(n, ctypes.byref(wsb)), "tgl_shard_unpermute_workspace")
    ws = torch.empty(max(wsb.value, 1), dtype=torch.uint8, device=dev)
    nnz = nbr_in.numel()
    off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    nbr = torch.empty(nnz, dtype=torch.int32, device=dev)
    eid = torch.empty(nnz, dtype=torch.int32, device=dev)
    dt = torch.empty(nnz, dtype=torch.float32, device=dev)
    _rc(_L.tgl_shard_unpermute(_ptr(perm), n, _ptr(counts_in), _ptr(nbr_in), _ptr(eid_in), _ptr(dt_in), _ptr(off),
                               _ptr(nbr), _ptr(eid), _ptr(dt), _ptr(ws), wsb.value, _stream(stream)),
        "tgl_shard_unpermute")
    return off, nbr, eid, dt


def shard_bucket(roots: torch.Tensor, splits: torch.Tensor, world: int, stream=None):
    """tgl_shard_bucket: stable permutation (int32) of roots by owner shard + per-shard counts."""
    roots = _cuda(roots, torch.int32, "roots")
    splits = _cuda(splits, torch.int64, "splits")
    n = roots.numel()
    wsb = ctypes.c_size_t()
    _rc(_L.tgl_shard_bucket_workspace(n, int(world), ctypes.byref(wsb)), "tgl_shard_bucket_workspace")
    ws = torch.empty(max(wsb.value, 1), dtype=torch.uint8, device=roots.device)
    perm = torch.empty(max(n, 1), dtype=torch.int32, device=roots.device)
    counts = torch.empty(int(world), dtype=torch.int64, device=roots.device)
    _rc(_L.tgl_shard_bucket(_ptr(roots), n, _ptr(splits), int(world), _ptr(perm), _ptr(counts), _ptr(ws),
                            wsb.value, _stream(stream)), "tgl_shard_bucket")
    return perm[:n], counts


# ----------------------------------------------------------------------------- node-sharded mode
def tcsr_indptr(src: torch.Tensor, dst: torch.Tensor, ts: torch.Tensor, *, n_nodes: int, add_reverse: bool,
                stream=None) -> torch.Tensor:
    """tgl_tcsr_indptr: the full graph's indptr only (validation + degree scan), e.g. to choose the
    edge-balanced node ranges of the node-sharded mode."""
    src = _cuda(src, torch.int32, "src")
    dst = _cuda(dst, torch.int32, "dst")
    ts = _cuda(ts, torch.float32, "ts")
    indptr = torch.empty(n_nodes + 1, dtype=torch.int64, device=src.device)
    b = ctypes.c_size_t()
    _rc(_L.tgl_tcsr_indptr_workspace(src.numel(), int(n_nodes), ctypes.byref(b)), "tgl_tcsr_indptr_workspace")
    ws = torch.empty(max(b.value, 1), dtype=torch.uint8, device=src.device)
    _rc(_L.tgl_tcsr_indptr(_ptr(src), _ptr(dst), _ptr(ts), src.numel(), int(n_nodes), int(add_reverse), _ptr(indptr),
                           _ptr(ws), b.value, _stream(stream)), "tgl_tcsr_indptr")
    return indptr


def build_range(src: torch.Tensor, dst: torch.Tensor, ts: torch.Tensor, eid: Optional[torch.Tensor] = None, *,
                n_nodes: int, add_reverse: bool, node_lo: int, node_hi: int, n_local_stored: int,
                with_index: bool = True, stream=None) -> TCSR:
    """tgl_tcsr_build_range: the T-CSR of the nodes [node_lo, node_hi) only (node base = node_lo)."""
    src = _cuda(src, torch.int32, "src")
    dst = _cuda(dst, torch.int32, "dst")
    ts = _cuda(ts, torch.float32, "ts")
    if eid is not None:
        eid = _cuda(eid, torch.int32, "eid")
    dev = src.device
    nl, es = int(node_hi) - int(node_lo), int(n_local_stored)
    indptr = torch.empty(nl + 1, dtype=torch.int64, device=dev)
    nbr = torch.empty(max(es, 1), dtype=torch.int32, device=dev)
    ts_out, ts_storage = _ts_buffer(max(es, 1), dev)
    eid_out = torch.empty(max(es, 1), dtype=torch.int32, device=dev)
    ib = aux_bytes(es, nl) if with_index else 0
    index = torch.empty(ib, dtype=torch.uint8, device=dev) if with_index else None
    b = ctypes.c_size_t()
    _rc(_L.tgl_tcsr_build_range_workspace(src.numel(), int(n_nodes), int(add_reverse), int(node_lo), int(node_hi), es,
                                          ctypes.byref(b)), "tgl_tcsr_build_range_workspace")
    ws = torch.empty(max(b.value, 1), dtype=torch.uint8, device=dev)
    h = ctypes.c_void_p()
    _rc(_L.tgl_tcsr_build_range(_ptr(src), _ptr(dst), _ptr(ts), _ptr(eid), src.numel(), int(n_nodes), int(add_reverse),
                                int(node_lo), int(node_hi), es, _ptr(indptr), _ptr(nbr), _ptr(ts_storage),
                                _ptr(eid_out), _ptr(index), ib, _ptr(ws), b.value, _stream(stream), ctypes.byref(h)),
        "tgl_tcsr_build_range")
    del ws
    g = TCSR(indptr, nbr[:es], ts_out[:es], eid_out[:es], nl, h, index, ts_storage)
    g.node_lo = int(node_lo)
    return g


def nccl_id() -> bytes:
    """tgl_shard_nccl_id: a fresh NCCL unique id (call on one rank, broadcast to the others)."""
    buf = (ctypes.c_char * _lib.NCCL_ID_BYTES)()
    _rc(_L.tgl_shard_nccl_id(buf), "tgl_shard_nccl_id")
    return bytes(buf)


class ShardGroup:
    """tgl_shard_group: an in-process group of ranks (threads of this process) for the node-sharded
    sampler, exchanging by device copies (tests and single-device runs)."""

    def __init__(self, world: int):
        self.world = int(world)
        h = ctypes.c_void_p()
        _rc(_L.tgl_shard_group_create(self.world, ctypes.byref(h)), "tgl_shard_group_create")
        self._h = h

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _L is not None:
            _L.tgl_shard_group_destroy(h)


class ShardSampler:
    """One rank of the node-sharded sampler (tgl_shard_create + tgl_sample_sharded): `local` holds
    the lists of nodes [splits[rank], splits[rank+1]) (tcsr with node base, e.g. build_range);
    exactly one transport: `nccl_id` (bytes of nccl_id() shared by all ranks: NCCL, one process
    per GPU) or `group` (ShardGroup: ranks on threads of this process).  run() is collective."""

    def __init__(self, local: TCSR, splits: Sequence[int], rank: int, world: int, max_roots: int,
                 fanouts: Sequence[int], strategy="most_recent", n_snapshots: int = 1,
                 snapshot_len: float = math.inf, *, nccl_id: Optional[bytes] = None,
                 group: Optional[ShardGroup] = None):
        self.local, self.group = local, group
        self.fanouts = [int(k) for k in fanouts]
        self.L, self.S = len(self.fanouts), int(n_snapshots)
        self.strategy = _strategy(strategy)
        self.snapshot_len = float(snapshot_len)
        self.max_roots = int(max_roots)
        sp = (ctypes.c_int64 * (int(world) + 1))(*[int(x) for x in splits])
        idb = None if nccl_id is None else ctypes.create_string_buffer(bytes(nccl_id), _lib.NCCL_ID_BYTES)
        h = ctypes.c_void_p()
        _rc(_L.tgl_shard_create(local.handle, sp, int(rank), int(world), idb,
                                None if group is None else group._h, ctypes.byref(h)), "tgl_shard_create")
        self._h = h
        self._fan = (ctypes.c_int32 * self.L)(*self.fanouts)
        rc_ = (ctypes.c_int64 * self.L)()
        ec_ = (ctypes.c_int64 * self.L)()
        wsb = ctypes.c_size_t()
        _rc(_L.tgl_sample_capacity(self.max_roots, self.L, self._fan, self.S, self.strategy, self.snapshot_len, rc_, ec_,
                                   ctypes.byref(wsb)), "tgl_sample_capacity")
        self.roots_cap, self.edges_cap = list(rc_), list(ec_)
        self.blocks = _alloc_blocks(local.nbr.device, self.roots_cap, self.edges_cap, self.L, self.S)
        self._c_blocks = _c_blocks(self.blocks, self.roots_cap, self.edges_cap, self.S)

    def run(self, roots: torch.Tensor, root_ts: torch.Tensor, *, seed: int = 0, root_key_base: int = 0,
            stream=None) -> List[Block]:
        roots = _cuda(roots, torch.int32, "roots")
        root_ts = _cuda(root_ts, torch.float32, "root_ts")
        n = roots.numel()
        if n > self.max_roots or root_ts.numel() < n:
            raise ValueError(f"{n} roots > max_roots {self.max_roots} or root_ts too short")
        _rc(_L.tgl_sample_sharded(self._h, _ptr(roots), _ptr(root_ts), n, self.L, self._fan, self.strategy, self.S,
                                  self.snapshot_len, int(seed) & 0xFFFFFFFFFFFFFFFF,
                                  int(root_key_base) & 0xFFFFFFFFFFFFFFFF, self._c_blocks, _stream(stream)),
            "tgl_sample_sharded")
        return self.blocks

    def gather(self, ids: torch.Tensor, local_tables: Sequence[torch.Tensor],
               outs: Optional[Sequence[torch.Tensor]] = None, stream=None) -> List[torch.Tensor]:
        """tgl_shard_gather (collective): rows of global nodes `ids` from tables sharded like the
        T-CSR; local_tables[j] = this rank's rows [n_local, ...] (a K-slot ring: [n_local, K, ...])."""
        ids = _cuda(ids, torch.int32, "ids")
        n = ids.numel()
        arr, res = (_lib.GatherTable * len(local_tables))(), []
        for j, t in enumerate(local_tables):
            if not (t.is_cuda and t.is_contiguous()):
                raise TypeError("local tables must be contiguous CUDA tensors")
            rb = t.element_size() * int(np.prod(t.shape[1:], dtype=np.int64))
            o = outs[j] if outs is not None else torch.empty((n,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            res.append(o)
            arr[j] = _lib.GatherTable(t.data_ptr(), t.shape[0], rb, o.data_ptr())
        _rc(_L.tgl_shard_gather(self._h, _ptr(ids), n, arr, len(local_tables), _stream(stream)), "tgl_shard_gather")
        return res

    def state_write(self, ids: torch.Tensor, ts: torch.Tensor, pairs, *, K: int = 1,
                    pos: Optional[torch.Tensor] = None, ts_table: Optional[torch.Tensor] = None, stream=None) -> None:
        """tgl_shard_state_write (collective): pairs = [(rows [n, ...], local table [n_local * K, ...])];
        pos / ts_table: this rank's local cursors [n_local] / times [n_local * K]."""
        ids = _cuda(ids, torch.int32, "ids")
        n = ids.numel()
        ts = _cuda(ts, torch.float32, "ts")
        arr = (_lib.StateTable * max(len(pairs), 1))()
        for j, (rows, table) in enumerate(pairs):
            if not (rows.is_cuda and table.is_cuda and rows.is_contiguous() and table.is_contiguous()):
                raise TypeError("state rows / tables must be contiguous CUDA tensors")
            rb = rows.element_size() * int(np.prod(rows.shape[1:], dtype=np.int64))
            arr[j] = _lib.StateTable(rows.data_ptr() if n else None, rb, table.data_ptr())
        if pos is not None:
            pos = _cuda(pos, torch.int32, "pos")
        if ts_table is not None:
            ts_table = _cuda(ts_table, torch.float32, "ts_table")
        _rc(_L.tgl_shard_state_write(self._h, _ptr(ids), _ptr(ts), n, int(K), _ptr(pos), _ptr(ts_table), arr, len(pairs),
                                     _stream(stream)), "tgl_shard_state_write")

    def stats(self):
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _rc(_L.tgl_shard_stats(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)), "tgl_shard_stats")
        return {"bytes_sent": a.value, "bytes_recv": b.value, "host_syncs": c.value}

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _L is not None:
            _L.tgl_shard_destroy(h)
