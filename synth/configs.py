"""The five paper-shaped synthetic workloads C1-C5 (BASELINE.json configs).

Inputs only -- no sampler arithmetic.  Every random quantity is a counter-based integer hash
of (config seed, stream id, element index), evaluated with int64 torch ops whose products
stay below 2^63, so the SAME bits come out on CPU and on GPU, chunk by chunk, in any order.
Skewed distributions use inverse-CDF tables built once in float64 numpy and then applied as
integer thresholds (searchsorted), again device-independent.

Shapes (Table 3; readings R#16-R#19 of DESIGN.md):
  C1 Wikipedia-shaped  9,227 nodes (8,227 users + 1,000 items), 157,474 edges, t in [0, 2.7e6]
  C2 Reddit-shaped    10,984 nodes (10,000 + 984), 672,447 edges, t in [0, 2.7e6]
  C3 LastFM-shaped     1,980 nodes (980 + 1,000), 1,293,103 edges, t in [0, 1.3e8] + tables
  C4 GDELT-shaped     16,682 actors, 191,290,882 edges, 15-minute ticks 0..1.8e5, Zipf(1.2) hubs
  C5 MAG-shaped      121,000,000 papers, 1,300,000,000 citations (+reverse), years 0..120
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np
import torch

M32 = 0xFFFFFFFF
_C1, _C2 = 0x7FEB352D, 0x2C1B3C6D          # odd multipliers < 2^31 (products fit in int64)
_GOLD = 0x9E3779B1


def _mix32(x: torch.Tensor) -> torch.Tensor:
    x = x ^ (x >> 16)
    x = (x * _C1) & M32
    x = x ^ (x >> 15)
    x = (x * _C2) & M32
    return x ^ (x >> 16)


def hash_u32(idx: torch.Tensor, seed: int, stream: int) -> torch.Tensor:
    """Uniform 32-bit value for each int64 index (0 <= idx < 2^62), as int64 in [0, 2^32)."""
    k = ((seed * 0x632BE5AB) ^ (stream * _GOLD)) & M32
    hi = _mix32(((idx >> 32) ^ k) & M32)
    return _mix32(((idx & M32) + hi + k) & M32)


def uniform_int(idx, seed, stream, n: int) -> torch.Tensor:
    """Integer in [0, n) (n < 2^31): (u32 * n) >> 32."""
    return (hash_u32(idx, seed, stream) * int(n)) >> 32


def _thresholds(pmf: np.ndarray) -> np.ndarray:
    cdf = np.cumsum(pmf / pmf.sum())
    thr = np.floor(cdf * 2.0**32).astype(np.int64)
    thr[-1] = 2**32
    return thr


def zipf_thresholds(n: int, s: float) -> np.ndarray:
    r = np.arange(1, n + 1, dtype=np.float64)
    return _thresholds(r ** (-s))


def table_draw(idx, seed, stream, thr: torch.Tensor) -> torch.Tensor:
    """Inverse-CDF draw: first r with u < thr[r]."""
    return torch.searchsorted(thr, hash_u32(idx, seed, stream), right=True)


def hash_f32(idx, seed, stream) -> torch.Tensor:
    """Exactly representable float32 in [-1, 1): (u >> 8) * 2^-23 - 1."""
    return ((hash_u32(idx, seed, stream) >> 8).to(torch.float64) * 2.0**-23 - 1.0).to(torch.float32)


@dataclass
class Workload:
    name: str
    n_nodes: int
    n_edges: int
    add_reverse: bool
    fanouts: List[int]
    strategy: str
    n_snapshots: int
    snapshot_len: float
    batch: int
    seed: int
    t_max: float
    bipartite_split: Optional[int] = None   # first item id for bipartite graphs (negatives drawn >= it)
    tables: Dict[str, tuple] = field(default_factory=dict)  # name -> (rows, cols) fp32 gather tables
    sampler_seed: int = 42

    @property
    def n_logical(self) -> int:
        return self.n_edges * (2 if self.add_reverse else 1)

    @property
    def n_roots_epoch(self) -> int:
        return 3 * self.n_edges


CONFIGS: Dict[str, Workload] = {
    "C1": Workload("wikipedia-shaped", 9_227, 157_474, True, [10], "most_recent", 1, math.inf, 600,
                   0x54474C00 + 1, 2.7e6, bipartite_split=8_227),
    "C2": Workload("reddit-shaped", 10_984, 672_447, True, [10, 10], "uniform", 1, math.inf, 600,
                   0x54474C00 + 2, 2.7e6, bipartite_split=10_000),
    "C3": Workload("lastfm-shaped", 1_980, 1_293_103, True, [10], "most_recent", 1, math.inf, 600,
                   0x54474C00 + 3, 1.3e8, bipartite_split=980,
                   tables={"memory": (1_980, 100), "mem_ts": (1_980, 1), "mailbox": (1_980, 428),
                           "mail_ts": (1_980, 1), "edge_feat": (1_293_103, 128)}),
    "C4": Workload("gdelt-shaped", 16_682, 191_290_882, False, [10, 10], "uniform", 1, math.inf, 4_000,
                   0x54474C00 + 4, 1.8e5),
    "C5": Workload("mag-shaped", 121_000_000, 1_300_000_000, True, [10], "most_recent", 3, 5.0, 4_000,
                   0x54474C00 + 5, 120.0),
    # DySAT's sampler workload of Table 4 on the C1 graph --
    # 2-layer uniform within 3 dynamic snapshots of 10,000 s; exercises reading R#3
    "C6": Workload("wikipedia-dysat", 9_227, 157_474, True, [10, 10], "uniform", 3, 10_000.0, 600,
                   0x54474C00 + 1, 2.7e6, bipartite_split=8_227),
}


def scaled(cfg: Workload, n_nodes: int, n_edges: int) -> Workload:
    """Same recipe at a smaller size (parity tests the oracle finishes in seconds)."""
    import dataclasses
    split = None
    if cfg.bipartite_split is not None:
        split = max(1, int(round(n_nodes * cfg.bipartite_split / cfg.n_nodes)))
        split = min(split, n_nodes - 1)
    tables = {k: ((n_nodes if r == cfg.n_nodes else n_edges), c) for k, (r, c) in cfg.tables.items()}
    return dataclasses.replace(cfg, n_nodes=n_nodes, n_edges=n_edges, bipartite_split=split, tables=tables)


# ----------------------------------------------------------------------------- edge streams
def _bipartite_chunk(cfg: Workload, lo: int, hi: int, dev) -> tuple:
    """User -> item interactions (C1-C3): Zipf(1.1) users, 80% repeat of one of 5 favourite items
    per user (stateless stand-in for repeat affinity), else Zipf(1.1) items; integer timestamps
    t_i = floor(i * (t_max+1) / E), non-decreasing with runs of equal times (ties)."""
    s = cfg.seed
    n_users = cfg.bipartite_split
    n_items = cfg.n_nodes - n_users
    i = torch.arange(lo, hi, dtype=torch.int64, device=dev)
    uthr = torch.from_numpy(zipf_thresholds(n_users, 1.1)).to(dev)
    ithr = torch.from_numpy(zipf_thresholds(n_items, 1.1)).to(dev)
    # Zipf rank -> id through a fixed hash order so hubs are spread over the id space
    user = (table_draw(i, s, 1, uthr) * 2_654_435_761) % n_users
    fav = (_mix32((user * 5 + uniform_int(i, s, 2, 5)) & M32) % n_items)
    other = (table_draw(i, s, 3, ithr) * 1_000_003) % n_items
    item = torch.where(hash_u32(i, s, 4) < int(0.8 * 2**32), fav, other)
    src = user
    dst = n_users + item
    ts = _sorted_times(i, cfg, dev)
    return src.to(torch.int32), dst.to(torch.int32), ts


def _sorted_times(i: torch.Tensor, cfg: Workload, dev) -> torch.Tensor:
    """Non-decreasing integer times over [0, t_max] for stream positions i (order-preserving)."""
    E = cfg.n_edges
    T = int(cfg.t_max)
    base = (i * (T + 1)) // E                      # monotone in i
    return base.to(torch.float32)


def _gdelt_chunk(cfg: Workload, lo: int, hi: int, dev) -> tuple:
    """Actor -> actor events (C4): Zipf(1.2) endpoints over 16,682 actors, 15-minute ticks
    0..1.8e5 (~1,060 events per tick -> heavy ties)."""
    s = cfg.seed
    V = cfg.n_nodes
    i = torch.arange(lo, hi, dtype=torch.int64, device=dev)
    thr = torch.from_numpy(zipf_thresholds(V, 1.2)).to(dev)
    src = (table_draw(i, s, 1, thr) * 2_654_435_761) % V
    dst = (table_draw(i, s, 2, thr) * 40_503 + 7) % V
    ts = _sorted_times(i, cfg, dev)
    return src.to(torch.int32), dst.to(torch.int32), ts


def _mag_year_table(cfg: Workload):
    years = int(cfg.t_max) + 1
    w = np.exp(0.05 * np.arange(years))
    cnt = np.floor(w / w.sum() * cfg.n_nodes).astype(np.int64)
    cnt[-1] += cfg.n_nodes - cnt.sum()
    start = np.zeros(years + 1, dtype=np.int64)
    np.cumsum(cnt, out=start[1:])
    q = 8.0 / 9.0                                     # geometric lag, mean 8 years
    lag_thr = _thresholds((1 - q) * q ** np.arange(years))
    return start, lag_thr


def feistel_perm(x: torch.Tensor, n: int, seed: int) -> torch.Tensor:
    """Bijection of [0, n) (n <= 2^30): 4-round Feistel on 2 x h bits (2^2h < 4n) with cycle
    walking (follows the permutation's cycle from x until it re-enters [0, n); terminates because
    the cycle contains x itself)."""
    h = max(1, ((max(n - 1, 1)).bit_length() + 1) // 2)
    hm = (1 << h) - 1

    def rounds(y):
        L, R = y >> h, y & hm
        for r in range(4):
            k = ((seed * 0x5851F42D) ^ (r * _GOLD)) & M32
            L, R = R, L ^ (_mix32((R ^ k) & M32) & hm)
        return (L << h) | R
    y = rounds(x)
    while True:
        bad = y >= n
        if not bool(bad.any()):
            return y
        y = torch.where(bad, rounds(y), y)


def _mag_chunk(cfg: Workload, lo: int, hi: int, dev) -> tuple:
    """Paper -> cited paper (C5): papers in year order, paper counts growing ~e^{0.05 y}; edge i is
    reference slot of citing paper p = floor(i V / E) (10-11 references each), at the citing year
    (P:L355); cited year = citing year - geometric lag (mean 8 y, clamped at 0); within the year a
    product-of-3-uniforms index (heavy-tailed in-degree).  Ids are Feistel-permuted."""
    s = cfg.seed
    V, E = cfg.n_nodes, cfg.n_edges
    start_np, lag_np = _mag_year_table(cfg)
    start = torch.from_numpy(start_np).to(dev)
    lag_thr = torch.from_numpy(lag_np).to(dev)
    i = torch.arange(lo, hi, dtype=torch.int64, device=dev)
    p = (i * V) // E
    year = torch.searchsorted(start, p, right=True) - 1
    lag = table_draw(i, s, 1, lag_thr)
    cy = torch.clamp(year - lag, min=0)
    n_y = start[cy + 1] - start[cy]
    idx = (n_y * hash_u32(i, s, 2)) >> 32
    idx = (idx * hash_u32(i, s, 3)) >> 32
    idx = (idx * hash_u32(i, s, 4)) >> 32
    cited = start[cy] + idx
    src = feistel_perm(p, V, s)
    dst = feistel_perm(cited, V, s)
    return src.to(torch.int32), dst.to(torch.int32), year.to(torch.float32)


_CHUNKERS = {"C1": _bipartite_chunk, "C2": _bipartite_chunk, "C3": _bipartite_chunk, "C4": _gdelt_chunk,
             "C5": _mag_chunk, "C6": _bipartite_chunk}


def edge_chunk(key: str, cfg: Workload, lo: int, hi: int, device="cpu"):
    """Edges [lo, hi) of config `key` (scaled or full): (src int32, dst int32, ts float32)."""
    return _CHUNKERS[key](cfg, lo, hi, torch.device(device))


def edges(key: str, cfg: Workload, device="cpu", chunk: int = 1 << 26):
    """The whole chronological stream on `device`, generated chunk by chunk."""
    E = cfg.n_edges
    dev = torch.device(device)
    src = torch.empty(E, dtype=torch.int32, device=dev)
    dst = torch.empty(E, dtype=torch.int32, device=dev)
    ts = torch.empty(E, dtype=torch.float32, device=dev)
    for lo in range(0, E, chunk):
        hi = min(E, lo + chunk)
        s, d, t = edge_chunk(key, cfg, lo, hi, dev)
        src[lo:hi], dst[lo:hi], ts[lo:hi] = s, d, t
    return src, dst, ts


# ----------------------------------------------------------------------------- roots (R#16, R#17)
def roots(cfg: Workload, src: torch.Tensor, dst: torch.Tensor, ts: torch.Tensor, first_root: int,
          n_roots: int, edge_offset: int = 0):
    """Roots [first_root, first_root + n_roots) of the root stream (src_i, dst_i, neg_i) at ts_i.

    src/dst/ts may be a window of the stream starting at edge `edge_offset`.  neg_i is uniform over
    the destination side: the item range for bipartite graphs, all nodes otherwise.
    """
    dev = src.device
    r = torch.arange(first_root, first_root + n_roots, dtype=torch.int64, device=dev)
    e = r // 3
    which = r % 3
    le = e - edge_offset
    if cfg.bipartite_split is not None:
        lo, n = cfg.bipartite_split, cfg.n_nodes - cfg.bipartite_split
    else:
        lo, n = 0, cfg.n_nodes
    neg = lo + uniform_int(e, cfg.seed, 9, n)
    node = torch.where(which == 0, src[le].to(torch.int64), torch.where(which == 1, dst[le].to(torch.int64), neg))
    return node.to(torch.int32), ts[le].clone()


def batch_edges(cfg: Workload, src: torch.Tensor, dst: torch.Tensor, ts: torch.Tensor, first_root: int,
                n_roots: int):
    """The mini-batch in TGL's own form ("600 positive and 600 negative edges"): the positive
    edges (src_i, dst_i, ts_i) covering roots [first_root, first_root + n_roots) of the root stream
    and their negative destinations neg_i (R#17) -- e0 = first_root // 3 and int32 / float32 arrays
    of the edges e0 .. (first_root + n_roots - 1) // 3.  roots() of the same range = their expansion."""
    e0, e1 = first_root // 3, (first_root + n_roots - 1) // 3 + 1
    e = torch.arange(e0, e1, dtype=torch.int64, device=src.device)
    if cfg.bipartite_split is not None:
        lo, n = cfg.bipartite_split, cfg.n_nodes - cfg.bipartite_split
    else:
        lo, n = 0, cfg.n_nodes
    neg = (lo + uniform_int(e, cfg.seed, 9, n)).to(torch.int32)
    return e0, src[e0:e1].clone(), dst[e0:e1].clone(), neg, ts[e0:e1].clone()


def tables(cfg: Workload, device="cpu") -> Dict[str, torch.Tensor]:
    """Gather sources for C3: node memory, mem_ts, mailbox (K=1, 428 wide, R#18), mail_ts, edge
    features (128-d, random as the paper does for LastFM, L428).  Exact float32 values."""
    out = {}
    dev = torch.device(device)
    for j, (name, (rows, cols)) in enumerate(sorted(cfg.tables.items())):
        idx = torch.arange(rows * cols, dtype=torch.int64, device=dev)
        out[name] = hash_f32(idx, cfg.seed, 100 + j).reshape(rows, cols) if cols > 1 else \
            hash_f32(idx, cfg.seed, 100 + j).abs().mul_(float(cfg.t_max)).reshape(rows)
    return out


def relevant_substream(src: torch.Tensor, dst: torch.Tensor, ts: torch.Tensor, nodes: torch.Tensor,
                       n_nodes: int, add_reverse: bool, chunk: int = 1 << 27):
    """Edges of the stream that can own a logical edge of one of `nodes`, in stream order, with
    their original indices as eids: (src, dst, ts, eid) numpy arrays.  Input selection for the
    restricted oracle on billion-edge configs (the oracle then applies its own owner filter)."""
    keep = torch.zeros(n_nodes, dtype=torch.bool, device=src.device)
    keep[nodes.long()] = True
    parts = []
    for lo in range(0, src.numel(), chunk):
        hi = min(src.numel(), lo + chunk)
        s, d = src[lo:hi].long(), dst[lo:hi].long()
        m = keep[s] | keep[d] if add_reverse else keep[s]
        idx = torch.nonzero(m).flatten()
        parts.append((s[idx].int().cpu(), d[idx].int().cpu(), ts[lo:hi][idx].cpu(), (idx + lo).int().cpu()))
    cat = [torch.cat([p[j] for p in parts]).numpy() if parts else np.zeros(0) for j in range(4)]
    return cat[0], cat[1], cat[2], cat[3], keep.cpu().numpy().astype(np.uint8)
