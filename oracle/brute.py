"""Brute-force sampler over the whole logical edge stream -- TEST INFRASTRUCTURE.

The bottom of the test pyramid (SURVEY 8(c) "What pins each part"): no T-CSR, no
binary search, no pointer.  For each root it scans every logical edge of the stream
and keeps those with owner == v and L <= ts < U ("scan all edges with ts < t",
north_star), in stream order (= the stable, chronological order of P:L256), then
selects by the strategy definition.  It has its own Philox4x32-10
(pure Python integers, written from Salmon et al. SC'11), independent of
``tgl_oracle.c``.  Small inputs only: O(|E|) numpy work per root.
"""
from __future__ import annotations

import math
from typing import List

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


def philox(ctr, key):
    c = [int(x) & MASK for x in ctr]
    k0, k1 = int(key[0]) & MASK, int(key[1]) & MASK
    for rnd in range(10):
        if rnd:
            k0, k1 = (k0 + W0) & MASK, (k1 + W1) & MASK
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        c = [((p1 >> 32) ^ c[1] ^ k0) & MASK, p1 & MASK, ((p0 >> 32) ^ c[3] ^ k1) & MASK, p0 & MASK]
    return c


def logical_stream(src, dst, ts, eid, add_reverse: bool):
    """Logical edges in stream order (R#19): j = i, or 2i (forward) and 2i+1 (reverse)."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    ts = np.asarray(ts, dtype=np.float32)
    eid = np.arange(len(src), dtype=np.int64) if eid is None else np.asarray(eid, dtype=np.int64)
    if not add_reverse:
        return src, dst, ts, eid
    owner = np.empty(2 * len(src), dtype=np.int64)
    nbr = np.empty_like(owner)
    owner[0::2], owner[1::2] = src, dst
    nbr[0::2], nbr[1::2] = dst, src
    return owner, nbr, np.repeat(ts, 2), np.repeat(eid, 2)


def floyd(c: int, k: int, seed: int, layer: int, snapshot: int, rk: int) -> List[int]:
    """Floyd's uniform k-subset of range(c); draw j = word j % 4 of the Philox block at counter
    j // 4 (R#5, R#6)."""
    picks: List[int] = []
    key = (seed & MASK, (seed >> 32) & MASK)
    for j in range(k):
        m = c - k + j
        x = philox((j // 4, (layer << 16) | snapshot, rk & MASK, (rk >> 32) & MASK), key)[j % 4]
        r = (x * (m + 1)) >> 32
        picks.append(m if r in picks else r)
    return sorted(picks)


def with_replacement(c: int, k: int, seed: int, layer: int, snapshot: int, rk: int) -> List[int]:
    """k independent uniform draws from range(c), draw j as in Floyd (R#24, R#6), sorted."""
    key = (seed & MASK, (seed >> 32) & MASK)
    return sorted((philox((j // 4, (layer << 16) | snapshot, rk & MASK, (rk >> 32) & MASK), key)[j % 4] * c) >> 32
                  for j in range(k))


def sample(src, dst, ts, eid, *, n_nodes: int, add_reverse: bool, roots, root_ts, fanouts,
           strategy: int, n_snapshots: int = 1, snapshot_len: float = math.inf, seed: int = 0,
           root_key_base: int = 0, hop_time: str = "edge", replacement: bool = False, dedup: bool = False,
           edge_valid=None):
    """Returns blocks[l*S+s] = list over roots of lists of (nbr, eid, dt, ts_edge)."""
    owner, nbr, tsl, eidl = logical_stream(src, dst, ts, eid, add_reverse)
    f32 = np.float32
    tsv = f32(snapshot_len)
    L, S = len(fanouts), n_snapshots
    blocks = [None] * (L * S)
    for s in range(S):
        # (node, t, key, lo) per root of the current layer
        cur = [(int(v), f32(t), (root_key_base + i) & 0xFFFFFFFFFFFFFFFF, None)
               for i, (v, t) in enumerate(zip(roots, root_ts))]
        for l in range(L):
            k = fanouts[l]
            out, nxt = [], []
            for (v, t, rk, lo_in) in cur:
                if not (0 <= v < n_nodes) or not np.isfinite(t):
                    out.append([])
                    continue
                if l == 0:
                    U = t if s == 0 else f32(t - f32(f32(s) * tsv))
                    Lo = f32(t - f32(f32(s + 1) * tsv))
                else:
                    U = t
                    Lo = lo_in if lo_in is not None else f32(-np.inf)
                ok = (owner == v) & (tsl >= Lo) & (tsl < U)
                if edge_valid is not None:  # R#28: invalid edges are not candidates
                    ev = np.asarray(edge_valid, dtype=np.uint64)
                    ok &= ((ev[eidl.astype(np.int64) >> 5] >> (eidl.astype(np.uint64) & np.uint64(31))) & np.uint64(1)) == 1
                cand = np.nonzero(ok)[0]
                c = len(cand)
                if strategy == 0:
                    sel = cand[max(0, c - k):]
                elif replacement:
                    sel = cand[with_replacement(c, k, seed, l, s, rk)] if c else cand
                elif c <= k:
                    sel = cand
                else:
                    sel = cand[floyd(c, k, seed, l, s, rk)]
                row = []
                for j, p in enumerate(sel):
                    row.append((int(nbr[p]), int(eidl[p]), f32(t - tsl[p]), f32(tsl[p])))
                    nxt.append((int(nbr[p]), f32(tsl[p]) if hop_time == "edge" else t,
                                (rk * k + j) & 0xFFFFFFFFFFFFFFFF,
                                Lo if math.isfinite(snapshot_len) else None))
                out.append(row)
            blocks[l * S + s] = out
            if dedup:  # R#27: distinct (node, time bits) in first-appearance order, first key wins
                seen, uniq = set(), []
                for (v, t, rk, lo) in nxt:
                    if (v, np.float32(t).view(np.uint32).item()) not in seen:
                        seen.add((v, np.float32(t).view(np.uint32).item()))
                        uniq.append((v, t, rk, lo))
                nxt = uniq
            cur = nxt
    return blocks


def tcsr(src, dst, ts, eid, *, n_nodes: int, add_reverse: bool):
    """T-CSR via numpy's stable argsort of owners (a library sort, not a counting sort)."""
    owner, nbr, tsl, eidl = logical_stream(src, dst, ts, eid, add_reverse)
    order = np.argsort(owner, kind="stable")
    indptr = np.zeros(n_nodes + 1, dtype=np.int64)
    np.cumsum(np.bincount(owner, minlength=n_nodes), out=indptr[1:])
    return dict(indptr=indptr, nbr=nbr[order].astype(np.int32), ts=tsl[order].astype(np.float32),
                eid=eidl[order].astype(np.int32))
