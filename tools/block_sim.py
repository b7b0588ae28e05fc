"""Host simulation (not a benchmark): random 128-B lines per C5 root for a node-major block layout
(header + records in 128-B aligned per-node blocks), one-pass search.  DESIGN.md section 8 "Next".
usage: python tools/block_sim.py <scale_div> <n_roots>"""
import sys, numpy as np
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from synth import configs as C
div = int(sys.argv[1]); n_roots = int(sys.argv[2])
base = C.CONFIGS["C5"]; cfg = C.scaled(base, base.n_nodes // div, base.n_edges // div)
src, dst, ts = C.edges("C5", cfg)
g = oracle.build(src.numpy(), dst.numpy(), ts.numpy(), n_nodes=cfg.n_nodes, add_reverse=True)
indptr, T = g["indptr"], g["ts"]
starts = np.linspace(0, cfg.n_roots_epoch - 4000, 32).astype(np.int64)
per = n_roots // 32; rs, rt = [], []
for s0 in starts:
    r, t = C.roots(cfg, src, dst, ts, int(s0), per); rs.append(r.numpy()); rt.append(t.numpy())
rs, rt = np.concatenate(rs), np.concatenate(rt)
k, S, tsl = 10, 3, np.float32(5.0)
def lb(a, b, x):
    while a < b:
        m = (a + b) // 2
        if T[m] < x: a = m + 1
        else: b = m
    return a
res = {}
for HB, RB in ((16, 12), (16, 16), (64, 12), (64, 16)):
  tot = 0
  for v, t in zip(rs.tolist(), rt.tolist()):
    t = np.float32(t); lo, hi = int(indptr[v]), int(indptr[v + 1])
    x = [t] + [np.float32(t - np.float32(np.float32(j) * tsl)) for j in range(1, S + 1)]
    cut = [lb(lo, hi, xj) for xj in x]
    sel = []
    for b in range(S):
        a, e = cut[b + 1], cut[b]; tk = min(k, e - a); sel += list(range(e - tk, e))
    # block: header HB bytes at offset 0 (128-aligned), record j at HB + RB*j; ideal search (no probe cost
    # beyond lines that hold the cut neighbours: ts[c-1], ts[c])
    lines = {0}
    for c in cut:
        for q in (c - 1, c):
            if lo <= q < hi: lines.add((HB + RB * (q - lo)) // 128)
    for q in sel: lines.add((HB + RB * (q - lo)) // 128)
    tot += len(lines)
  res[(HB, RB)] = tot / len(rs)
print(res)
