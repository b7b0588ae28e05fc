"""Random-access cost model of the C5 sampler layouts (host simulation, not a benchmark).

On C5 the sampler is bound by the number of random DRAM requests per root (DESIGN.md section 4:
~30-34 G requests/s whatever the request size up to 128 B).  This script builds a scaled C5 graph
with the oracle, draws roots spread over the epoch like bench.py, and counts per root the distinct
64-B / 128-B lines each layout touches:

  node   the node record (64 B: 14 fences, 128 B: 30 fences)
  probe  ts lines read by the cut searches inside the fence gaps (4-B ts array)
  recs   slot-record lines of the selected slots (16-B or 12-B records)

usage: python tools/atom_sim.py [scale_div] [n_roots]
"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (host tool: the oracle builds the T-CSR)
from synth import configs as C  # noqa: E402


def fence_pos(lo, d, j, F):
    return lo + (j * (d - 1)) // (F - 1)


def lower_bound(ts, a, b, x):
    while a < b:
        m = (a + b) // 2
        if ts[m] < x:
            a = m + 1
        else:
            b = m
    return a


def probes(ts, a, b, x, lines, line_bytes):
    """Lines of the 4-B ts array touched by a binary search for x in [a, b)."""
    while a < b:
        m = (a + b) // 2
        lines.add((m * 4) // line_bytes)
        if ts[m] < x:
            a = m + 1
        else:
            b = m
    return a


def main():
    div = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    n_roots = int(sys.argv[2]) if len(sys.argv) > 2 else 60_000
    base = C.CONFIGS["C5"]
    cfg = C.scaled(base, base.n_nodes // div, base.n_edges // div)
    src, dst, ts = C.edges("C5", cfg)
    g = oracle.build(src.numpy(), dst.numpy(), ts.numpy(), n_nodes=cfg.n_nodes, add_reverse=True)
    indptr, T = g["indptr"], g["ts"]
    starts = np.linspace(0, cfg.n_roots_epoch - 4000, 32).astype(np.int64)
    per = n_roots // 32
    rs, rt = [], []
    for s0 in starts:
        r, t = C.roots(cfg, src, dst, ts, int(s0), per)
        rs.append(r.numpy())
        rt.append(t.numpy())
    rs, rt = np.concatenate(rs), np.concatenate(rt)
    k, S, tsl = 10, 3, np.float32(5.0)
    acc = {}

    def add(key, v):
        acc[key] = acc.get(key, 0) + v

    deg = []
    for v, t in zip(rs.tolist(), rt.tolist()):
        t = np.float32(t)
        lo, hi = int(indptr[v]), int(indptr[v + 1])
        d = hi - lo
        deg.append(d)
        x = [t] + [np.float32(t - np.float32(np.float32(j) * tsl)) for j in range(1, S + 1)]
        cut = [lower_bound(T, lo, hi, xj) for xj in x]
        sel = []
        for b in range(S):
            a, e = cut[b + 1], cut[b]
            sel += list(range(max(a, e - k), e))
        add("edges", len(sel))
        add("nonzero", 1 if sel else 0)
        for F in (14, 30):
            for LB in (64, 128):
                lines = set()
                if d and T[lo] < t:
                    for xj in x:
                        if d <= F:
                            continue
                        fs = [T[fence_pos(lo, d, j, F)] for j in range(F)]
                        m = sum(1 for f in fs if f < xj)
                        ga = fence_pos(lo, d, m - 1, F) + 1 if m else lo
                        gb = fence_pos(lo, d, m, F) if m < F else hi
                        probes(T, ga, gb, xj, lines, LB)
                add(f"probe_F{F}_L{LB}", len(lines))
        for rec in (16, 12, 8):
            for LB in (64, 128):
                add(f"recs_R{rec}_L{LB}", len({(p * rec) // LB for p in sel}))
        # node-major blocks: 64-B header then the node's 16-B records, block 64-B aligned
        # (header line + record lines; the header line also holds records 0..? -> none here)
    n = len(rs)
    deg = np.array(deg)
    print(f"C5 / {div}: {cfg.n_nodes} nodes, {cfg.n_edges} edges; {n} roots; mean degree {deg.mean():.1f}, "
          f"edges/root {acc['edges'] / n:.2f}, nonzero roots {acc['nonzero'] / n:.3f}")
    for key in sorted(acc):
        if key in ("edges", "nonzero"):
            continue
        print(f"  {key:16s} {acc[key] / n:.3f} lines/root")
    q = np.percentile(deg, [10, 25, 50, 75, 90, 99])
    print("  degree percentiles 10/25/50/75/90/99:", q)


if __name__ == "__main__":
    main()
