"""Host census (not a benchmark): scattered DRAM requests per C5 root under the product layout and
under alternative node-record encodings.  1/div-scale C5 (same per-node structure: ~10.7 references
per paper at its own year, citations later), roots from chunks spread over the epoch like bench.py.

Counts per root (upper bounds on L2-missing requests: no L2 reuse across roots is modelled, except
that a root whose node equals the previous root of the same kind reuses the node record):
  rec     the 64-byte node record
  probe   distinct 64-byte ts atoms touched by the fence-gap binary searches (product)
  copy    distinct 128-byte lines of 12-byte slot records holding the selected slots
Alternatives:
  runs<R> node record = {lo, hi} + the first slot of each of the node's last R distinct-time runs
          (exact cuts when every searched time falls inside the covered runs, else fences+probes)
usage: python tools/census_c5.py <div> <n_roots>
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from synth import configs as C  # noqa: E402

div = int(sys.argv[1]) if len(sys.argv) > 1 else 100
n_roots = int(sys.argv[2]) if len(sys.argv) > 2 else 200_000
base = C.CONFIGS["C5"]
cfg = C.scaled(base, base.n_nodes // div, base.n_edges // div)
src, dst, ts = C.edges("C5", cfg)
g = oracle.build(src.numpy(), dst.numpy(), ts.numpy(), n_nodes=cfg.n_nodes, add_reverse=True)
indptr, T = g["indptr"].astype(np.int64), g["ts"]
starts = np.linspace(0, cfg.n_roots_epoch - 4000, 25).astype(np.int64)
per = n_roots // 25
rs, rt, kind = [], [], []
for s0 in starts:
    s0 = int(s0) // 3 * 3
    r, t = C.roots(cfg, src, dst, ts, s0, per)
    rs.append(r.numpy()); rt.append(t.numpy()); kind.append(np.arange(per) % 3)
rs, rt, kind = np.concatenate(rs), np.concatenate(rt), np.concatenate(kind)
k, S, tsl, F = 10, 3, np.float32(5.0), 14


def fence_pos(lo, d, j):
    return lo + (j * (d - 1)) // (F - 1)


def runs_of(lo, hi):
    """first slots of the distinct-time runs of the node's list"""
    if hi <= lo:
        return np.zeros(0, np.int64)
    tt = T[lo:hi]
    chg = np.nonzero(np.diff(tt) != 0)[0] + 1
    return np.concatenate([[0], chg]) + lo


tot = {"rec": 0, "probe": 0, "copy": 0, "sel_roots": 0, "early": 0}
by_kind = np.zeros((3, 3))
alt = {R: 0 for R in (4, 6, 8, 12)}
fvar = {(14, 16): 0, (14, 64): 0, (28, 64): 0, (56, 64): 0}
prev = [-1, -1, -1]
nr = len(rs)
for v, t, kd in zip(rs.tolist(), rt.tolist(), kind.tolist()):
    t = np.float32(t)
    lo, hi = int(indptr[v]), int(indptr[v + 1])
    d = hi - lo
    x = [t] + [np.float32(t - np.float32(np.float32(j) * tsl)) for j in range(1, S + 1)]
    rec = 0 if prev[kd] == v else 1
    prev[kd] = v
    tot["rec"] += rec
    by_kind[kd, 0] += rec
    early = d > 0 and T[lo] < t
    cuts = [int(lo + np.searchsorted(T[lo:hi], xj, side="left")) for xj in x]
    atoms = set()
    if early:
        tot["early"] += 1
        fences = [T[fence_pos(lo, d, j)] if d > 0 else np.inf for j in range(F)]
        for xj in x:
            m = int(np.sum(np.array(fences) < xj))
            a = fence_pos(lo, d, m - 1) + 1 if m else lo
            b = fence_pos(lo, d, m) if m < F else hi
            while a < b:
                mid = a + (b - a) // 2
                atoms.add(mid // 16)
                if T[mid] < xj:
                    a = mid + 1
                else:
                    b = mid
    tot["probe"] += len(atoms)
    if early:
        for (FF, APA) in fvar:
            at2 = set()
            fp = [lo + (j * (d - 1)) // (FF - 1) for j in range(FF)]
            fv = np.array([T[q] for q in fp])
            for xj in x:
                m = int(np.sum(fv < xj))
                a = fp[m - 1] + 1 if m else lo
                b = fp[m] if m < FF else hi
                while a < b:
                    mid = a + (b - a) // 2
                    at2.add(mid // APA)
                    if T[mid] < xj:
                        a = mid + 1
                    else:
                        b = mid
            fvar[(FF, APA)] += len(at2)
    by_kind[kd, 1] += len(atoms)
    lines8 = set()
    for bb in range(S):
        a, e = cuts[bb + 1], cuts[bb]
        tk = min(k, e - a)
        for q in range(e - tk, e):
            lines8.add(q * 8 // 128)
    tot["copy8"] = tot.get("copy8", 0) + len(lines8)
    lines = set()
    for bb in range(S):
        a, e = cuts[bb + 1], cuts[bb]
        tk = min(k, e - a)
        for q in range(e - tk, e):
            lines.add(q * 12 // 128)
    tot["copy"] += len(lines)
    by_kind[kd, 2] += len(lines)
    tot["sel_roots"] += bool(lines)
    # alternative: exact runs for the node's last R runs (or all if fewer); cut exact if x lies in
    # [ts of the first covered run, +inf) -- else the product's fence search for that cut
    if early:
        rr = runs_of(lo, hi)
        for R in alt:
            cov = rr[-R:] if len(rr) > R else rr
            first_cov_t = T[cov[0]]
            # a cut x is exact when x > ts of the slot before the first covered run or all runs covered
            need = set()
            if len(rr) > R:
                fences = [T[fence_pos(lo, d, j)] for j in range(F)]
                for xj in x:
                    if xj > first_cov_t:
                        continue
                    m = int(np.sum(np.array(fences) < xj))
                    a = fence_pos(lo, d, m - 1) + 1 if m else lo
                    b = fence_pos(lo, d, m) if m < F else hi
                    while a < b:
                        mid = a + (b - a) // 2
                        need.add(mid // 16)
                        if T[mid] < xj:
                            a = mid + 1
                        else:
                            b = mid
            alt[R] += len(need)
print(f"C5 1/{div}: {nr} roots, early {tot['early'] / nr:.3f}, selecting {tot['sel_roots'] / nr:.3f}")
print(f"per root: node record {tot['rec'] / nr:.3f}, probes {tot['probe'] / nr:.3f}, copy lines {tot['copy'] / nr:.3f}")
for kd, name in enumerate(("src", "dst", "neg")):
    n = np.sum(kind == kd)
    print(f"  {name}: rec {by_kind[kd, 0] / n:.3f} probe {by_kind[kd, 1] / n:.3f} copy {by_kind[kd, 2] / n:.3f}")
print(f"copy lines with 8-byte records {tot['copy8'] / nr:.3f}")
for FF, v in fvar.items():
    print(f"fences {FF[0]}, {FF[1]} slots per probe atom: probes per root {v / nr:.3f}")
for R, v in alt.items():
    print(f"runs{R}: probes per root {v / nr:.3f}")
