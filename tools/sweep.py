"""Tuning sweep for the sampler on one config (default C5): times tgl_sample per setting.

python tools/sweep.py [--config C5] [--roots 1048576] [--reps 10]
Settings are the library's experiment knobs (TGL_NO_STAGE, TGL_NO_RECS, TGL_NO_INDEX) plus the
no-aux (plain binary search) handle.  Prints one JSON line per setting.
"""
import argparse
import itertools
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
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--only", default="", help="comma list k=v of one setting to run (e.g. for ncu)")
ap.add_argument("--settings", default="", help="JSON list of env dicts (aux handle) to run instead")
args = ap.parse_args()
cfg = C.CONFIGS[args.config]
src, dst, ts = C.edges(args.config, cfg, device="cuda")
g = tgl.build(src, dst, ts, n_nodes=cfg.n_nodes, add_reverse=cfg.add_reverse)
g_plain = tgl.wrap(g.indptr, g.nbr, g.ts, g.eid, with_index=False)
torch.cuda.empty_cache()
n_steps = args.reps + 3
starts = [int(x) // cfg.batch * cfg.batch for x in torch.linspace(0, cfg.n_roots_epoch - args.roots, n_steps)]
chunks = [C.roots(cfg, src, dst, ts, s0, args.roots) for s0 in starts]
del src, dst
torch.cuda.empty_cache()


def run(handle, env):
    for k in [k for k in os.environ if k.startswith("TGL_") and k != "TGL_LIB_PATH"]:
        os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in env.items()})
    smp = tgl.Sampler(handle, args.roots, cfg.fanouts, cfg.strategy, cfg.n_snapshots, cfg.snapshot_len)
    for j in range(3):
        smp.run(*chunks[j], seed=cfg.sampler_seed, root_key_base=starts[j])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for j in range(3, n_steps):
        smp.run(*chunks[j], seed=cfg.sampler_seed, root_key_base=starts[j])
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.reps
    edges = 0
    for j in range(3, n_steps):
        blocks = smp.run(*chunks[j], seed=cfg.sampler_seed, root_key_base=starts[j])
        edges += sum(int(x.nnz_dev.item()) for x in blocks)
    return ms, edges / args.reps


settings = [("aux", {}), ("aux", {"TGL_NO_STAGE": 1}), ("aux", {"TGL_NO_RECS": 1}),
            ("aux", {"TGL_NO_INDEX": 1}), ("plain", {})]
if args.settings:
    settings = [("aux", e) for e in json.loads(args.settings)]
if args.only:
    env = dict(kv.split("=") for kv in args.only.split(","))
    settings = [("plain" if env.pop("handle", "aux") == "plain" else "aux", env)]
for name, env in settings:
    ms, edges = run(g if name == "aux" else g_plain, env)
    print(json.dumps({"handle": name, **env, "ms": round(ms, 4), "roots_per_s": args.roots / ms * 1e3,
                      "edges_per_s": edges / ms * 1e3}), flush=True)
