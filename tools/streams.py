"""Does running independent tgl_sample calls on several CUDA streams overlap their kernels?

python tools/streams.py [--config C5] [--roots 1048576] [--streams 1 2 3 4]
Each stream has its own Sampler (workspace + outputs); steps are distributed round-robin.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_14883_b200 as tgl  # noqa: E402
from synth import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--roots", type=int, default=1 << 20)
ap.add_argument("--steps", type=int, default=16)
ap.add_argument("--streams", type=int, nargs="+", default=[1, 2, 3, 4])
args = ap.parse_args()
cfg = C.CONFIGS[args.config]
src, dst, ts = C.edges(args.config, cfg, device="cuda")
g = tgl.build(src, dst, ts, n_nodes=cfg.n_nodes, add_reverse=cfg.add_reverse)
torch.cuda.empty_cache()
starts = [int(x) // cfg.batch * cfg.batch for x in torch.linspace(0, cfg.n_roots_epoch - args.roots, args.steps + 4)]
chunks = [C.roots(cfg, src, dst, ts, s0, args.roots) for s0 in starts]
del src, dst
torch.cuda.empty_cache()
for ns in args.streams:
    streams = [torch.cuda.Stream() for _ in range(ns)]
    smps = [tgl.Sampler(g, args.roots, cfg.fanouts, cfg.strategy, cfg.n_snapshots, cfg.snapshot_len) for _ in range(ns)]
    for j in range(4):  # warm-up
        with torch.cuda.stream(streams[j % ns]):
            smps[j % ns].run(*chunks[j], seed=cfg.sampler_seed, root_key_base=starts[j])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for s in streams:
        s.wait_event(a)
    for j in range(args.steps):
        with torch.cuda.stream(streams[j % ns]):
            smps[j % ns].run(*chunks[4 + j], seed=cfg.sampler_seed, root_key_base=starts[4 + j])
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    print(json.dumps({"streams": ns, "ms_per_call": round(ms, 4), "roots_per_s": args.roots / ms * 1e3}), flush=True)
