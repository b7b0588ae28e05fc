"""Experiment (not a bench number): does running the window kernel of one root chunk concurrently
with the copy kernel of another raise C5 throughput?  Splits the bench step (8,192,000 roots) into
P pieces, each a tgl_sample call with its own Sampler, issued round-robin on Q streams; compares the
device time with one call over the whole step.  Outputs are compared by digest with the one-call run.

python tools/concur.py [--pieces 2,4,8] [--streams 2]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2203_14883_b200 as tgl  # noqa: E402
from synth import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--pieces", default="1,2,4,8")
ap.add_argument("--streams", type=int, default=2)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
cfg = C.CONFIGS[args.config]
B = cfg.batch
n = 2048 * B
src, dst, ts = C.edges(args.config, cfg, device="cuda")
g = tgl.build(src, dst, ts, n_nodes=cfg.n_nodes, add_reverse=cfg.add_reverse)
torch.cuda.empty_cache()
starts = bench.chunk_starts(cfg.n_roots_epoch, n, args.reps + 2, B)
chunks = [C.roots(cfg, src, dst, ts, s0, n) for s0 in starts]
del src, dst, ts
torch.cuda.empty_cache()
L, S = len(cfg.fanouts), cfg.n_snapshots
streams = [torch.cuda.Stream() for _ in range(args.streams)]

for P in [int(x) for x in args.pieces.split(",")]:
    m = n // P
    smps = [tgl.Sampler(g, m, cfg.fanouts, cfg.strategy, S, cfg.snapshot_len) for _ in range(P)]

    def run(j):
        r, t = chunks[j]
        cur = torch.cuda.current_stream()
        for q in range(P):
            st = streams[q % len(streams)]
            st.wait_stream(cur)
        for q in range(P):
            st = streams[q % len(streams)]
            with torch.cuda.stream(st):
                smps[q].run(r[q * m:(q + 1) * m], t[q * m:(q + 1) * m], seed=cfg.sampler_seed,
                            root_key_base=starts[j] + q * m)
        for st in streams:
            cur.wait_stream(st)

    for j in range(2):
        run(j)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for j in range(2, args.reps + 2):
        run(j)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.reps
    run(args.reps + 1)
    torch.cuda.synchronize()
    edges = sum(int(x.nnz_dev.item()) for s in smps for x in s.blocks)
    dig = [bench.gpu_batch_digests(tgl, s.blocks, m, B, L, S) for s in smps]
    d = np.concatenate(dig, axis=1)
    print(json.dumps({"pieces": P, "streams": args.streams, "ms_per_step": round(ms, 4),
                      "G_edges_per_s": round(edges / ms / 1e6, 2),
                      "digest_xor": int(np.bitwise_xor.reduce(d.reshape(-1)))}), flush=True)
