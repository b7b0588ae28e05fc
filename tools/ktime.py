"""Per-kernel device time of tgl_sample on one config under several env settings (torch.profiler /
CUPTI kernel records; not a bench number).  Also reports the fraction of roots whose first edge
is not earlier than the root time (the upper bound of the first-time skip, tsindex.cuh).

python tools/ktime.py [--config C5] [--roots 8192000] [--reps 5] [--settings '[{}, {"TGL_NO_SKIP": 1}]']
"""
import argparse
import json
import os
import sys
from collections import defaultdict

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_14883_b200 as tgl  # noqa: E402
from synth import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--roots", type=int, default=2048 * 4000)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--settings", default='[{}]')
args = ap.parse_args()
cfg = C.CONFIGS[args.config]
src, dst, ts = C.edges(args.config, cfg, device="cuda")
g = tgl.build(src, dst, ts, n_nodes=cfg.n_nodes, add_reverse=cfg.add_reverse)
torch.cuda.empty_cache()
n_steps = args.reps + 2
starts = [int(x) // cfg.batch * cfg.batch for x in torch.linspace(0, cfg.n_roots_epoch - args.roots, n_steps)]
chunks = [C.roots(cfg, src, dst, ts, s0, args.roots) for s0 in starts]
del src, dst
torch.cuda.empty_cache()
r, t = chunks[-1]
lo = g.indptr[r.long()]
hi = g.indptr[r.long() + 1]
first = torch.where(hi > lo, g.ts[lo.clamp(max=g.ts.numel() - 1)], torch.full_like(t, float("inf")))
print(json.dumps({"roots": int(r.numel()), "first_ge_t": float((first >= t).float().mean()), "codec": g.codec}),
      flush=True)

for env in json.loads(args.settings):
    for k in [k for k in os.environ if k.startswith("TGL_") and k != "TGL_LIB_PATH"]:
        os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in env.items()})
    smp = tgl.Sampler(g, args.roots, cfg.fanouts, cfg.strategy, cfg.n_snapshots, cfg.snapshot_len)
    for j in range(2):
        smp.run(*chunks[j], seed=cfg.sampler_seed, root_key_base=starts[j])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for j in range(2, n_steps):
        smp.run(*chunks[j], seed=cfg.sampler_seed, root_key_base=starts[j])
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.reps
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for j in range(2, n_steps):
            smp.run(*chunks[j], seed=cfg.sampler_seed, root_key_base=starts[j])
        torch.cuda.synchronize()
    per = defaultdict(float)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            name = e.name.split("<")[0].split("(")[0].replace("void ", "").replace("tgl::", "")
            per[name] += e.device_time_total / args.reps
    out_blocks = smp.run(*chunks[-1], seed=cfg.sampler_seed, root_key_base=starts[-1])
    edges = sum(int(x.nnz_dev.item()) for x in out_blocks)
    digest = 0  # output fingerprint: settings must agree bit for bit
    for x in out_blocks:
        off, nbr, eid, dt, _ = x.trimmed()
        for a in (off.view(torch.int32), nbr, eid, dt.view(torch.int32)):
            w = torch.arange(1, a.numel() + 1, device=a.device, dtype=torch.int64)
            digest = (digest * 1000003 + int(((a.to(torch.int64) & 0xFFFFFFFF) * w).sum().item())) % (1 << 61)
    print(json.dumps({"env": env, "digest": digest, "ms_per_call": round(ms, 4), "G_edges_per_s": round(edges / ms / 1e6, 2),
                      "kernels_us": {k: round(v, 1) for k, v in sorted(per.items(), key=lambda x: -x[1])}}),
          flush=True)
