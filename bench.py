"""Benchmark: sampled temporal edges/s of TGL's sampler (Alg. 1) on B200, vs HBM roofline, vs oracle.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]

A step = one tgl_sample call over `--batches` consecutive mini-batches of the configuration's
root stream (epoch mode; per-batch calls are latency-bound), i.e. one pass of the
whole sampling path: window bounds, cut searches, selection, payload + dt, CSR offsets.  The
T-CSR is built once before timing (its time is reported as build_ms, excluded).  Steps are spread
evenly over the epoch's root stream, all distinct; the T-CSR (32 GB for C5) and the step inputs
exceed L2, so no flush is needed between steps.

N > 1 (torchrun, one process per GPU): every rank holds a replicated T-CSR (built from the same
seeded input) and samples its own batches (batch b -> rank b mod N): no collective on the data
path ("scaling": "weak"); the reporting all_reduce happens after the timed region.

--impl reference: the CPU oracle (oracle/, single thread) as the reference arm, same metric and
workload, each step a bounded sample of the workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import configs as C  # noqa: E402

METRIC = "sampled temporal edges/s"
UNIT = "edges/s"


# ----------------------------------------------------------------------------- helpers
def workload_name(key: str, cfg: C.Workload) -> str:
    """config.workload of every bench line (ours, node-sharded and the reference arm): one name per config."""
    return (f"{key} {cfg.name}: {cfg.n_nodes:,} nodes, {cfg.n_edges:,} edges"
            f"{' (+reverse)' if cfg.add_reverse else ''}, {len(cfg.fanouts)}-layer "
            f"{cfg.strategy} k={cfg.fanouts}, {cfg.n_snapshots} snapshot(s)"
            f"{'' if not math.isfinite(cfg.snapshot_len) else f' of {cfg.snapshot_len:g}'}")


def algorithmic_bytes(cfg: C.Workload, n_roots_per_layer, nnz_per_layer) -> int:
    """Bytes the method must move, element granularity.

    Per root of layer l: root read 8 B (l >= 1: + 4 B inherited L if S > 1), indptr pair 16 B,
    8 B per distinct cut (S+1 with finite t_s, else 1; l >= 1: 1 + finite L), offsets 8 B per block.
    Per sampled edge: read (nbr, eid, ts) 12 B + write (nbr, eid, dt) 12 B, + 4 B ts_edge if
    l < L-1.
    """
    L, S = len(cfg.fanouts), cfg.n_snapshots
    finite = math.isfinite(cfg.snapshot_len)
    total = 0
    for l in range(L):
        if l == 0:
            per_root = 8 + 16 + 8 * ((S + 1) if finite else 1) + 8 * S
        else:
            per_root = 8 + (4 if S > 1 else 0) + 16 + 8 * (2 if finite else 1) + 8
        per_edge = 24 + (4 if l < L - 1 else 0)
        total += per_root * n_roots_per_layer[l] + per_edge * nnz_per_layer[l]
    return int(total)


class ClockSampler:
    """Polls SM clock + throttle reasons with NVML from a thread during the timed region."""

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self.period = period_s
        self.ok = False
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)
        self._stop = threading.Event()

    _REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
                0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
                0x100: "display_clock_setting"}

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self._REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "note": getattr(self, "err", "no samples")}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def chunk_starts(n_total_roots: int, chunk: int, n_chunks: int, batch: int):
    span = max(0, n_total_roots - chunk)
    out = []
    for c in range(n_chunks):
        s = span * c // max(1, n_chunks - 1) if n_chunks > 1 else 0
        out.append(s // batch * batch)
    return out


def gather_bytes(cfg: C.Workload, n_roots: int, nnz: int) -> int:
    """Algorithmic bytes of the C3 gather: read + write of every gathered row; node
    tables for the roots and the sampled neighbours, edge features for the sampled eids."""
    node_row = sum(4 * cols for name, (rows, cols) in cfg.tables.items() if name != "edge_feat")
    edge_row = 4 * cfg.tables["edge_feat"][1]
    return 2 * ((n_roots + nnz) * node_row + nnz * edge_row)


def state_bytes(cfg: C.Workload, n_events: int) -> int:
    """Algorithmic bytes of the C3 state write (Fig. 2 step 6): per event read its id + time (8 B)
    and its new memory / mail rows, write them and the two timestamps into the node tables."""
    node_row = sum(4 * cols for name, (rows, cols) in cfg.tables.items() if name in ("memory", "mailbox"))
    return n_events * (8 + 2 * node_row + 2 * 4)


def chunk_events(s0: int, r: torch.Tensor, t: torch.Tensor):
    """The events of Fig. 2 step 6 in a root chunk: the positive-edge endpoints (src_i, dst_i at
    ts_i; root stream R#16 = (src_i, dst_i, neg_i) per edge), in batch order.  Input setup."""
    j = torch.arange(r.numel(), device=r.device)
    keep = ((s0 + j) % 3) != 2
    return r[keep].contiguous(), t[keep].contiguous()


def state_write_launches(tgl, cfg, K: int = 1) -> int:
    """Kernels of one tgl_state_write: keys + passes x (upsweep + 3 scan + downsweep) + slot + copy."""
    bits = max(1, int(cfg.n_nodes).bit_length())
    return 1 + 5 * max(1, (bits + 7) // 8) + 2 + (1 if K > 1 else 0)


def fused_spec(tabs):
    """Fused gather (tgl_fused_gather): the copy kernel writes each sampled edge's node rows (memory,
    mem_ts, mailbox, mail_ts) and edge-feature row; only the roots' rows take a separate gather."""
    return [(tabs["memory"], "node"), (tabs["mem_ts"], "node"), (tabs["mailbox"], "node"), (tabs["mail_ts"], "node"),
            (tabs["edge_feat"], "edge")]


def make_gather(tgl, cfg, sampler, dev, tabs=None, fused=False):
    """C3 data path of Fig. 2: step 2 -- memory, mem_ts, mailbox, mail_ts for the roots
    and sampled neighbours, edge features for the sampled eids (preallocated outputs, device-side
    counts) -- and step 6 -- the batch's events write their new memory (mem_ts) and mail (mail_ts)
    into the node tables (tgl_state_write, K = 1, R#25).  The new rows are the memory updater's /
    mail builder's outputs (model code, out of scope): resident synthetic rows stand in."""
    tabs = C.tables(cfg, device=dev) if tabs is None else tabs
    node_tabs = [tabs[k] for k in ("memory", "mem_ts", "mailbox", "mail_ts")]
    cap_r, cap_e = sampler.roots_cap[0], sampler.edges_cap[0]
    out_r = [torch.empty((cap_r,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev) for t in node_tabs]
    out_n = [] if fused else [torch.empty((cap_e,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev) for t in node_tabs]
    out_e = [] if fused else [torch.empty((cap_e, tabs["edge_feat"].shape[1]), dtype=torch.float32, device=dev)]
    gen = torch.Generator(device=dev)
    gen.manual_seed(cfg.seed)
    new_mem = torch.randn((cap_r, tabs["memory"].shape[1]), generator=gen, device=dev)
    new_mail = torch.randn((cap_r, tabs["mailbox"].shape[1]), generator=gen, device=dev)
    writer = tgl.StateWriter(cfg.n_nodes, cap_r, device=dev)

    marks = []  # (gather start, gather end / state start, state end) events of timed steps

    def run(roots, block, events=None, mark=False):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if mark else None
        if mark:
            ev[0].record()
        tgl.gather(roots, node_tabs, outs=out_r)
        if not fused:  # (fused: the sampler's copy kernel wrote the sampled edges' rows)
            tgl.gather(block.nbr, node_tabs, n_ids_dev=block.nnz_dev, outs=out_n)
            tgl.gather(block.eid, [tabs["edge_feat"]], n_ids_dev=block.nnz_dev, outs=out_e)
        if mark:
            ev[1].record()
        if events is not None:
            ids, ets = events
            n = ids.numel()
            writer(ids, ets, [(new_mem[:n], tabs["memory"]), (new_mail[:n], tabs["mailbox"]), (ets, tabs["mail_ts"])],
                   K=1, ts_table=tabs["mem_ts"])
        if mark:
            ev[2].record()
            marks.append(ev)
    run.marks = marks
    return run


def rank_chunks(n_epoch_roots: int, chunk: int, steps_total: int, world: int, rank: int, batch: int):
    """Root-sharded data parallelism: the steps_total * world chunks of `chunk` roots are spread
    evenly over the epoch and chunk c*world + r goes to rank r (batch-aligned, disjoint)."""
    starts = chunk_starts(n_epoch_roots, chunk, steps_total * world, batch)
    return [starts[c * world + rank] for c in range(steps_total)]


def measured_traffic(key: str, roots_per_step: float):
    """DRAM bytes per step of the sampler kernels from the committed ncu --set full capture
    (tools/ncu_traffic.py: dram__bytes_read.sum + dram__bytes_write.sum per root of the captured
    launches, x this step's roots).  TGL_TRAFFIC_JSON overrides the newest profiles/r*/traffic.json."""
    import glob
    path = os.environ.get("TGL_TRAFFIC_JSON")
    if not path:
        cands = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r*",
                                              "traffic.json")))
        path = cands[-1] if cands else None
    if not path or not os.path.exists(path):
        return None, None
    d = json.load(open(path)).get(key)
    if not d:
        return None, None
    src = (f"{os.path.relpath(path, os.path.dirname(os.path.abspath(__file__)))}: ncu --set full "
           f"({d['capture']}, {d['roots']:,} roots per launch), DRAM read + write of "
           f"{' + '.join(sorted(d['kernels']))} = {d['bytes_per_root']:.1f} B per root x roots per step")
    return d["bytes_per_root"] * roots_per_step, src


def measured_random_access(key: str, roots_per_step: float, kern_ms: float):
    """The sampler's binding resource on HBM-scale graphs: scattered DRAM requests (L2 misses).
    Requests per root from the committed ncu capture (lts__t_requests_srcunit_tex_lookup_miss of
    the sampler kernels), the peak request rate from tools/granule.cu in the same profiles dir."""
    import glob
    path = os.environ.get("TGL_TRAFFIC_JSON")
    if not path:
        cands = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "traffic.json")))
        path = cands[-1] if cands else None
    if not path or not os.path.exists(path):
        return None
    d = json.load(open(path)).get(key) or {}
    pk = os.path.join(os.path.dirname(path), "granule_peak.json")
    if "l2_read_miss_requests_per_root" not in d or not os.path.exists(pk):
        return None
    peak = json.load(open(pk))["peak_l2_read_miss_Greq_per_s"]
    rpr = d["l2_read_miss_requests_per_root"]
    achieved = rpr * roots_per_step / (kern_ms / 1e3) / 1e9
    return {"bound": "dram_random_requests", "requests_per_root": rpr, "achieved": achieved, "peak": peak,
            "unit": "G L2-missing read requests/s", "frac": achieved / peak,
            "source": f"{os.path.relpath(path, ROOT)} (ncu lts__t_requests_srcunit_tex_op_read_lookup_miss of the sampler "
                      f"kernels) / {os.path.relpath(pk, ROOT)} (tools/granule.cu: 4-byte reads at random lines of "
                      "32 GB)"}


def measured_shares(key: str):
    """Per-kernel DRAM bytes per root and share of the sampler kernels' time in the committed ncu
    capture (same file as measured_traffic) -- for comparing with the live step time."""
    import glob
    path = os.environ.get("TGL_TRAFFIC_JSON")
    if not path:
        cands = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r*",
                                              "traffic.json")))
        path = cands[-1] if cands else None
    if not path or not os.path.exists(path):
        return None
    d = json.load(open(path)).get(key)
    if not d:
        return None
    tot = sum(v["us"] for v in d["kernels"].values())
    return {k: {"ncu_us": v["us"], "share": v["us"] / tot, "dram_bytes_per_root": (v["dram_read"] + v["dram_write"])
                / d["roots"]} for k, v in d["kernels"].items()}


def reduce_report(edges: float, nbytes: float, ms: float, world: int, dev):
    """Reporting only (outside the timed region): sum of work over ranks, max of device time."""
    if world == 1:
        return float(edges), float(nbytes), float(ms)
    import torch.distributed as dist
    tot = torch.tensor([edges, nbytes], dtype=torch.float64, device=dev)
    mx = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(tot)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    return float(tot[0]), float(tot[1]), float(mx[0])


def setup_graph(key: str, cfg: C.Workload, dev):
    t0 = time.time()
    src, dst, ts = C.edges(key, cfg, device=dev)
    torch.cuda.synchronize(dev)
    gen_s = time.time() - t0
    return src, dst, ts, gen_s


# ----------------------------------------------------------------------------- node-sharded mode
def run_node_sharded(args):
    """SURVEY 8(e) node-sharded T-CSR through the C ABI: every rank computes the global degree scan
    (tgl_tcsr_indptr), takes the edge-balanced node range [splits[r], splits[r+1]) and builds ONLY
    that range (tgl_tcsr_build_range: ~E_s / N per rank); one NCCL communicator (tgl_shard_create,
    id broadcast through torch.distributed); each step is one collective tgl_sample_sharded over the
    rank's own root chunk: owner bucketing, NCCL all-to-all of counts / requests / replies, sampling
    on the owner's range, un-permute -- blocks bit-identical to the replicated mode (checked by
    per-batch digests against the oracle on the first timed chunk)."""
    import paper_2203_14883_b200 as tgl
    from paper_2203_14883_b200 import sharded as sh
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    key = args.config
    cfg = C.CONFIGS[key]
    B = cfg.batch
    L, S = len(cfg.fanouts), cfg.n_snapshots
    chunk = args.batches * B
    src, dst, ts, gen_s = setup_graph(key, cfg, dev)
    t0 = time.time()
    indptr = tgl.tcsr_indptr(src, dst, ts, n_nodes=cfg.n_nodes, add_reverse=cfg.add_reverse)
    splits = [int(x) for x in sh.edge_balanced_splits(indptr, world).cpu()]
    lo, hi = splits[rank], splits[rank + 1]
    n_local = int(indptr[hi] - indptr[lo])
    del indptr
    g = tgl.build_range(src, dst, ts, n_nodes=cfg.n_nodes, add_reverse=cfg.add_reverse, node_lo=lo, node_hi=hi,
                        n_local_stored=n_local)
    torch.cuda.synchronize(dev)
    build_s = time.time() - t0
    n_distinct = max(1, min(args.warmup + args.steps, args.distinct))
    mine = rank_chunks(cfg.n_roots_epoch, chunk, n_distinct, world, rank, B)
    chunks = [C.roots(cfg, src, dst, ts, s0, chunk) for s0 in mine]
    uid = [tgl.nccl_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    smp = tgl.ShardSampler(g, splits, rank, world, chunk, cfg.fanouts, cfg.strategy, S, cfg.snapshot_len,
                           nccl_id=uid[0])

    def step(j):
        r, t = chunks[j % n_distinct]
        return smp.run(r, t, seed=cfg.sampler_seed, root_key_base=mine[j % n_distinct])

    for w in range(args.warmup):
        step(w)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    st0 = smp.stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    with clocks:
        e0.record()
        for j in range(args.steps):
            step(args.warmup + j)
        e1.record()
        torch.cuda.synchronize(dev)
    st1 = smp.stats()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    # work (deterministic re-runs) + per-batch digests of every timed step
    edges, digests = 0, {}
    for j in range(args.steps):
        blocks = step(args.warmup + j)
        edges += sum(int(b.nnz_dev.item()) for b in blocks)
        digests[mine[(args.warmup + j) % n_distinct]] = gpu_batch_digests(tgl, blocks, chunk, B, L, S)
    # parity: the oracle's digests of this rank's first timed chunk
    s0 = mine[args.warmup % n_distinct]
    r0, t0_ = chunks[args.warmup % n_distinct]
    go, _ = oracle_graph(cfg, src, dst, ts, [r0])
    per_batch, _ = oracle_batches(go, cfg, r0.cpu().numpy(), t0_.cpu().numpy(), s0,
                                  max(1, host_info()["cores_available"] // max(1, world)))
    ok = bool(np.array_equal(oracle_batch_digests(per_batch, L * S), digests[s0]))
    del go, per_batch
    sent = float(st1["bytes_sent"] - st0["bytes_sent"])
    tot = torch.tensor([float(edges), sent, 0.0 if ok else 1.0], dtype=torch.float64, device=dev)
    mx = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    ms_max = float(mx[0])
    failed = tot[2].item() > 0 or tgl.check(g) != 0
    nv_peak = 900.0  # GB/s per direction per GPU over NVLink 5 (B200_PROFILING.md nominal)
    nv_rate = sent / (ms / 1e3) / 1e9 if ms > 0 else 0.0
    out = {"metric": METRIC, "value": None if failed else float(tot[0]) / (ms_max / 1e3), "unit": UNIT,
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": workload_name(key, cfg), "batch_roots": B, "batches_per_step": args.batches,
                      "roots_per_step_per_gpu": chunk,
                      "parallelism": f"node-sharded T-CSR over {world} rank(s) (tgl_tcsr_build_range), edge-balanced "
                                     "node ranges; tgl_sample_sharded: NCCL send/recv of counts, requests, replies",
                      "shard_nodes": hi - lo, "shard_edges": n_local,
                      "l2": "no flush: shard and per-step roots exceed L2"},
           "exchange": {"bytes_sent_per_step_per_rank": sent / args.steps,
                        "host_syncs_per_step": (st1["host_syncs"] - st0["host_syncs"]) / args.steps,
                        "nvlink_GBps_per_rank": nv_rate, "nvlink_peak_GBps": nv_peak, "nvlink_frac": nv_rate / nv_peak,
                        "note": "bytes to OTHER ranks only (none at N = 1: the exchange is a self-send)"},
           "parity": {"bit_exact": not failed, "against": "oracle per-batch FNV-1a digests, first timed chunk of "
                                                          "every rank", "checked_roots": chunk * world},
           # per call: the root keys + per chain bucketing (owner, upsweep, 3 scan, downsweep, counts), pack,
           # window + copy, reply counts; per block offsets->counts, un-permute (2 x 3 scan + counts + copy),
           # block sizes; per deeper chain the child keys (NCCL's own kernels not counted)
           "gpu_launches": args.steps * (1 + (11 + 10 * S) + (L - 1) * S * (11 + 10 + 1)),
           "clocks": clocks.summary(), "generate_s": gen_s, "build_s": build_s,
           "note": "the timed step includes the protocol's 2 host synchronisations per chain"}
    if failed:
        out["error"] = "parity failure or device error: no throughput reported"
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    if failed:
        sys.exit(1)


# ----------------------------------------------------------------------------- parity (oracle side)
def oracle_graph(cfg, src, dst, ts, root_tensors):
    """The oracle's T-CSR for the given layer-0 roots: restricted to their nodes (1 layer; the
    oracle's own count / fill passes over the stream sub-selected to those nodes), or the whole
    graph when deeper layers may reach any list.  Returns (T-CSR, build seconds)."""
    import oracle
    t0 = time.perf_counter()
    if len(cfg.fanouts) > 1:
        nodes = torch.arange(cfg.n_nodes, dtype=torch.int32, device=src.device)
    else:
        nodes = torch.cat([r for r in root_tensors])
    s_np, d_np, t_np, e_np, keep = C.relevant_substream(src, dst, ts, nodes, cfg.n_nodes, cfg.add_reverse)
    go = oracle.build_restricted(lambda: iter([(s_np, d_np, t_np, e_np, 0)]), n_nodes=cfg.n_nodes,
                                 add_reverse=cfg.add_reverse, keep=keep)
    return go, time.perf_counter() - t0


def oracle_batches(go, cfg, r_np, t_np, key0, n_threads, n_batches=None):
    """The oracle on consecutive batches of a root chunk (batch b: roots [b*B, (b+1)*B), key base
    key0 + b*B), in a thread pool (the oracle is stateless per root and its C call releases the
    GIL, so any thread count gives the same bits).  Returns (per-batch block lists, seconds)."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    B = cfg.batch
    nb = (len(r_np) + B - 1) // B if n_batches is None else n_batches
    strat = 0 if cfg.strategy == "most_recent" else 1

    def one(b):
        return oracle.sample(go, r_np[b * B:(b + 1) * B], t_np[b * B:(b + 1) * B], fanouts=cfg.fanouts, strategy=strat,
                             n_snapshots=cfg.n_snapshots, snapshot_len=cfg.snapshot_len, seed=cfg.sampler_seed,
                             root_key_base=key0 + b * B)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max(1, n_threads)) as ex:
        outs = list(ex.map(one, range(nb)))
    return outs, time.perf_counter() - t0


def concat_batches(per_batch, n_blocks):
    """Per-batch oracle blocks -> one block per (l, s) over all batches (offsets rebased), i.e. what
    a single many-batch tgl_sample call must write (epoch mode == per-batch mode, R#7)."""
    out = []
    for q in range(n_blocks):
        offs, base = [np.zeros(1, dtype=np.int64)], 0
        for bl in per_batch:
            o = bl[q]["offsets"]
            offs.append(o[1:] + base)
            base += int(o[-1])
        out.append({"offsets": np.concatenate(offs),
                    **{k: np.concatenate([bl[q][k] for bl in per_batch]) for k in ("nbr", "eid", "dt")}})
    return out


def compare_blocks(blocks, expected):
    """Element-by-element comparison (ids, eids, offsets; dt as bit patterns) of a GPU call's blocks
    with the oracle's.  Returns (ok, message of the first mismatch or None)."""
    for q, (b, e) in enumerate(zip(blocks, expected)):
        off, nbr, eid, dt, _ = b.trimmed()
        got = {"offsets": off.cpu().numpy(), "nbr": nbr.cpu().numpy(), "eid": eid.cpu().numpy(),
               "dt": dt.cpu().numpy().view(np.uint32)}
        want = dict(e, dt=e["dt"].view(np.uint32))
        for k in ("offsets", "nbr", "eid", "dt"):
            a, w = got[k], want[k]
            if a.shape != w.shape:
                return False, f"block {q} {k}: length {a.shape[0]} vs oracle {w.shape[0]}"
            bad = np.flatnonzero(a != w)
            if bad.size:
                return False, f"block {q} {k}[{bad[0]}] = {a[bad[0]]} vs oracle {w[bad[0]]} ({bad.size} differ)"
    return True, None


def gpu_batch_digests(tgl, blocks, n_roots, B, L, S):
    """tgl_block_digest of every (l, s) block, per batch of B layer-0 roots: uint64 [L*S, n_batches].
    Layer l >= 1 batch bounds = the parent block's offsets at the parent's bounds."""
    dev = blocks[0].offsets.device
    nb = (n_roots + B - 1) // B
    b0 = torch.clamp(torch.arange(nb + 1, dtype=torch.int64, device=dev) * B, max=n_roots)
    out = [None] * (L * S)
    for s in range(S):
        bounds = b0
        for l in range(L):
            q = l * S + s
            if l > 0:
                bounds = blocks[(l - 1) * S + s].offsets[bounds]
            out[q] = tgl.block_digest(blocks[q], bounds)
    return torch.stack(out).cpu().numpy().view(np.uint64)


def oracle_batch_digests(per_batch, n_blocks):
    import oracle
    return np.array([[oracle.block_digest(bl[q]) for bl in per_batch] for q in range(n_blocks)], dtype=np.uint64)


def host_info():
    """CPU model, logical cores available to this process and RAM of the host."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    ram = None
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                ram = round(int(line.split()[1]) / 2**20, 1)
                break
    except OSError:
        pass
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return {"cpu_model": model, "cores_available": cores, "ram_gib": ram}


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import paper_2203_14883_b200 as tgl
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # more ranks than GPUs (a launcher test on a 1-GPU box): ranks share the devices and the
    # reporting collectives run over gloo; the line says so ("oversubscribed") -- not a scaling number
    n_dev = max(1, torch.cuda.device_count())
    oversub = world > n_dev
    torch.cuda.set_device(local % n_dev)
    dev = torch.device("cuda", local % n_dev)
    cdev = torch.device("cpu") if oversub else dev  # device of the reporting collectives
    if world > 1:
        import torch.distributed as dist
        if oversub:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    key = args.config
    cfg = C.CONFIGS[key]
    B = cfg.batch
    M = args.batches
    chunk = M * B
    src, dst, ts, gen_s = setup_graph(key, cfg, dev)

    # T-CSR build (reported separately, excluded from the metric)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g = tgl.build(src, dst, ts, n_nodes=cfg.n_nodes, add_reverse=cfg.add_reverse)
    e1.record()
    torch.cuda.synchronize(dev)
    build_ms = e0.elapsed_time(e1)
    torch.cuda.empty_cache()

    # root chunks of this rank: chunk index c*world + rank, spread over the epoch
    # (at most --distinct different chunks, cycled: a chunk's footprint is GBs, far beyond L2)
    n_distinct = max(1, min(args.warmup + args.steps, args.distinct))
    mine = rank_chunks(cfg.n_roots_epoch, chunk, n_distinct, world, rank, B)
    chunks = [C.roots(cfg, src, dst, ts, s0, chunk) for s0 in mine]
    mine = [mine[j % n_distinct] for j in range(args.warmup + args.steps)]
    chunks = [chunks[j % n_distinct] for j in range(args.warmup + args.steps)]
    fused = bool(cfg.tables) and not args.separate_gather
    tabs = C.tables(cfg, device=dev) if fused else None
    sampler = tgl.Sampler(g, chunk, cfg.fanouts, cfg.strategy, cfg.n_snapshots, cfg.snapshot_len,
                          fused_gather=fused_spec(tabs) if fused else None)
    L, S = len(cfg.fanouts), cfg.n_snapshots
    launches_per_step = 2 * (1 + (L - 1) * S)  # window + copy kernel per chain (+1 memset, not ours)
    gather = make_gather(tgl, cfg, sampler, dev, tabs=tabs, fused=fused) if cfg.tables else None
    events = {}
    if gather is not None:
        # node tables by roots, node tables by nbr, edge features by eid (fused: roots + mail_ts); state write
        launches_per_step += (1 if fused else 3) + state_write_launches(tgl, cfg)
        for (r, t), s0 in zip(chunks, mine):
            if id(r) not in events:
                events[id(r)] = chunk_events(s0, r, t)

    def step(j, mark=False):
        r, t = chunks[j]
        blocks = sampler.run(r, t, seed=cfg.sampler_seed, root_key_base=mine[j])
        if gather is not None:
            gather(r, blocks[0], events[id(r)], mark=mark)
        return blocks

    for w in range(args.warmup):
        step(w)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    # a T-CSR (+ aux) that fits L2 would stay resident across steps: then a buffer larger than L2 is
    # written between timed steps and the time is the sum of the per-step event intervals
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    graph_bytes = g.indptr.numel() * 8 + g.n_stored * 28 + cfg.n_nodes * 64
    flush = graph_bytes < l2_bytes
    flush_buf = torch.empty(4 * l2_bytes, dtype=torch.uint8, device=dev) if flush else None
    clocks = ClockSampler(local)
    with clocks:
        t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        t_start.record()
        for j in range(args.steps):
            r, t = chunks[args.warmup + j]
            if flush:
                flush_buf.fill_(j & 0xFF)
            ev[j][0].record()
            step(args.warmup + j, mark=True)
            ev[j][1].record()
        t_end.record()
        torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms) if flush else t_start.elapsed_time(t_end)

    # digests of the LAST timed step's blocks as the timed call left them (before any re-run)
    n_last = chunks[args.warmup + args.steps - 1][0].numel()
    timed_last_digests = gpu_batch_digests(tgl, sampler.blocks, n_last, B, L, S)

    # work done per timed step (deterministic: re-run untimed and read the device counts) and the
    # per-batch digests of every timed batch, compared with the oracle's below
    edges_total, bytes_total, roots_total = 0, 0, 0
    digests_by_start = {}
    for j in range(args.steps):
        r, t = chunks[args.warmup + j]
        blocks = step(args.warmup + j)
        nr = [int(blocks[l * S].n_roots_dev.item()) for l in range(L)]
        nz = [sum(int(blocks[l * S + s].nnz_dev.item()) for s in range(S)) for l in range(L)]
        # per-layer roots over all S chains for l >= 1
        nr = [nr[0]] + [sum(int(blocks[l * S + s].n_roots_dev.item()) for s in range(S)) for l in range(1, L)]
        edges_total += sum(nz)
        roots_total += nr[0]
        bytes_total += algorithmic_bytes(cfg, nr, nz)
        if gather is not None:
            bytes_total += gather_bytes(cfg, nr[0], nz[0]) + state_bytes(cfg, events[id(r)][0].numel())
        digests_by_start[mine[args.warmup + j]] = gpu_batch_digests(tgl, blocks, r.numel(), B, L, S)
    rerun_same = bool(np.array_equal(digests_by_start[mine[args.warmup + args.steps - 1]], timed_last_digests))
    err = tgl.check(g)

    edges_all, bytes_all, total_ms_max = reduce_report(edges_total, bytes_total, total_ms, world, cdev)

    value = edges_all / (total_ms_max / 1e3)
    tcsr_bytes = g.indptr.numel() * 8 + g.n_stored * 12
    peak, peak_src = measured_peak_hbm()
    # dominant kernel = the sampler kernel (one launch per step for 1-layer configs); the per-step
    # events bracket tgl_sample = one small memset of the look-back state + the kernel(s)
    kern_ms = float(np.mean(step_ms))
    traffic, traffic_src = measured_traffic(key, roots_total / args.steps) if gather is None else (None, None)
    achieved = (bytes_total / args.steps) / (kern_ms / 1e3) / 1e9
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(key, cfg),
                   "batch_roots": B, "batches_per_step": M, "roots_per_step_per_gpu": chunk,
                   "parallelism": f"root-sharded dp{world}, replicated T-CSR",
                   **({"fused_gather": "tgl_fused_gather: edge rows written by the copy kernel"} if fused else {}),
                   "l2": (f"flushed: T-CSR + aux ({graph_bytes / 2**20:.0f} MiB) fit L2, so a {4 * l2_bytes >> 20} MiB "
                          "buffer is written between timed steps; time = sum of the per-step CUDA-event "
                          "intervals (flush excluded); the e2e leg is a host-fed pipeline, not flushed"
                          if flush else
                          "no flush: T-CSR and per-step roots exceed L2 (126 MB); "
                          f"{n_distinct} distinct root chunks cycled over the steps")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                     "kernels_ncu": measured_shares(key) if gather is None else None,
                     "random_access": measured_random_access(key, roots_total / args.steps, kern_ms)
                     if gather is None else None,
                     "kernel": (f"tgl_sample ({cfg.strategy}): window_kernel + copy_kernel"
                                + (" + tgl_gather (3 launches) + tgl_state_write" if gather is not None else "")
                                + ", timed together"),
                     "bytes_model": "SURVEY 8(d): per root 8+16+8*cuts+8*S, per edge 24 (+4 ts_edge if l<L-1)"
                                    + ("; gather: 2 x row bytes per gathered id; state write: 8 + 2 x (memory + mail "
                                       "row) + 8 B per event" if gather is not None else ""),
                     "algorithmic_bytes_per_step": bytes_total / args.steps,
                     "l2_resident": tcsr_bytes < l2_bytes,
                     "note": ("T-CSR + gather node tables fit the 126 MB L2 (flushed between steps, but the "
                              "re-reads inside a step hit L2): algorithmic bytes are mostly L2 traffic, so frac "
                              "vs the HBM peak is not meaningful here (SURVEY 8(d))")
                             if tcsr_bytes < l2_bytes else "T-CSR exceeds L2: HBM-bound random access"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks.summary(),
        "build_ms": build_ms, "generate_s": gen_s,
        # the T-CSR aux layout of this graph: the lossless time codec when the
        # graph has <= 127 distinct times (C5: publication years), 8-byte packed slot records
        "tcsr_layout": {"time_codes": g.codec["n_codes"], "packed_slot_records": g.codec["packed"]},
        "edges_per_step": edges_total / args.steps, "roots_per_step": roots_total / args.steps,
        "device_error": int(err),
        **({"oversubscribed": f"{world} ranks on {n_dev} GPU(s): launcher test, not a scaling number"}
           if oversub else {}),
    }

    if gather is not None and gather.marks and not fused:
        # Fig. 2 step 2 alone: the three gathers (node tables by roots and by sampled neighbours, edge
        # features by sampled eids) against the HBM peak, and the state write (step 6) beside it
        g_ms = sum(a.elapsed_time(b) for a, b, _ in gather.marks) / len(gather.marks)
        s_ms = sum(b.elapsed_time(c) for _, b, c in gather.marks) / len(gather.marks)
        gb = gather_bytes(cfg, roots_total // args.steps, int(edges_total // args.steps))
        node_row = sum(4 * cols for name, (rows, cols) in cfg.tables.items() if name != "edge_feat")
        edge_row = 4 * cfg.tables["edge_feat"][1]
        # HBM floor: every gathered row is written; of the reads only the edge features come from HBM
        # (the 4 MB node tables stay in L2)
        floor = (roots_total // args.steps + int(edges_total // args.steps)) * node_row \
            + 2 * int(edges_total // args.steps) * edge_row
        sb = state_bytes(cfg, int(np.mean([events[id(chunks[args.warmup + j][0])][0].numel() for j in range(args.steps)])))
        out["gather_roofline"] = {"bound": "hbm", "bytes_per_step": gb, "ms_per_step": g_ms,
                                  "achieved": gb / (g_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                                  "frac": gb / (g_ms / 1e3) / 1e9 / peak,
                                  "hbm_floor_bytes_per_step": floor,
                                  "frac_of_hbm_floor": floor / (g_ms / 1e3) / 1e9 / peak,
                                  "note": "tgl_gather x 3 (node tables by roots and by nbr, 660 MB edge-feature table "
                                          "by eid), CUDA events around the three launches of each timed step; bytes = "
                                          "read + write of every gathered row (the node tables themselves are L2-resident)"}
        out["state_write"] = {"bytes_per_step": sb, "ms_per_step": s_ms, "GBps": sb / (s_ms / 1e3) / 1e9}

    # per-batch mode (SURVEY 8(d) mode 1): one tgl_sample call per batch, replayed as a CUDA graph
    if not args.no_per_batch:
        mid = n_distinct // 2  # a chunk from the middle of the epoch (early batches have short histories)
        out["per_batch"] = per_batch(args, tgl, g, cfg, chunks[mid], mine[mid], dev, world, cdev=cdev)

    # end to end through the public API with host buffers (rank-local), copies inside the region
    if not args.no_e2e:
        gf = (lambda smp: make_gather(tgl, cfg, smp, dev, tabs=tabs, fused=fused)) if gather is not None else None
        # the mini-batches as TGL feeds them: positive edges + negatives (host), roots staged on the device
        by_start = {}
        for (r, _), s0 in zip(chunks, mine):
            if s0 not in by_start:
                by_start[s0] = C.batch_edges(cfg, src, dst, ts, s0, r.numel())
        bedges = [by_start[s0] for s0 in mine]
        out["e2e"] = e2e(args, tgl, sampler, chunks, mine, cfg, dev, world, gather_factory=gf, cdev=cdev,
                         events=events if gather is not None else None, batch_edges=bedges)
        out["e2e_root_arrays"] = e2e(args, tgl, sampler, chunks, mine, cfg, dev, world, gather_factory=gf, cdev=cdev,
                                     events=events if gather is not None else None)
        out["e2e_full_d2h"] = e2e(args, tgl, sampler, chunks, mine, cfg, dev, world, full_d2h=True, cdev=cdev,
                                  batch_edges=bedges)
        del by_start, bedges

    # parity gate (every rank, its own timed chunks) + CPU oracle baseline (rank 0, N = 1 only)
    out["parity"], cpu = parity_gate(args, cfg, tgl, sampler, src, dst, ts, chunks, mine, digests_by_start,
                                     rerun_same, world, want_cpu=world == 1 and not args.no_cpu_baseline)
    if cpu is not None:
        out["cpu_baseline"] = cpu
    failed = not out["parity"]["bit_exact"] or err != 0
    if world > 1:
        flag = torch.tensor([1.0 if failed else 0.0], device=cdev)
        torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MAX)
        failed = bool(flag.item())
    if failed:  # a run whose outputs do not match the oracle reports no throughput
        out["error"] = "parity failure or device error: no throughput reported"
        out["value_unverified"], out["value"] = out["value"], None
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    if failed:
        sys.exit(1)


def per_batch(args, tgl, g, cfg, chunk, key0, dev, world, n_graph=64, reps=10, cdev=None):
    """Latency mode: n_graph consecutive batches, one tgl_sample call each (batch b's roots, key base
    = its global root index), captured once as a CUDA graph and replayed; device time per batch =
    replay time / n_graph (CUDA events, max over ranks).  Edges counted from an eager re-run."""
    B = cfg.batch
    r, t = chunk
    n_graph = max(1, min(n_graph, r.numel() // B))
    smp = tgl.Sampler(g, B, cfg.fanouts, cfg.strategy, cfg.n_snapshots, cfg.snapshot_len)
    L, S = len(cfg.fanouts), cfg.n_snapshots

    def calls():
        for j in range(n_graph):
            smp.run(r[j * B:(j + 1) * B], t[j * B:(j + 1) * B], seed=cfg.sampler_seed, root_key_base=key0 + j * B)

    edges = 0
    for j in range(n_graph):  # eager pass: warm-up + the work count
        blocks = smp.run(r[j * B:(j + 1) * B], t[j * B:(j + 1) * B], seed=cfg.sampler_seed,
                         root_key_base=key0 + j * B)
        edges += sum(int(blocks[q].nnz_dev.item()) for q in range(L * S))
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        calls()  # warm-up on the capture stream
        torch.cuda.synchronize(dev)
        with torch.cuda.graph(graph, stream=side):
            calls()
    torch.cuda.synchronize(dev)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        graph.replay()
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    edges_all, _, ms_max = reduce_report(edges * reps, 0.0, ms, world, cdev or dev)
    launches = 2 * (1 + (L - 1) * S)
    return {"batch_roots": B, "batches_per_graph": n_graph, "replays": reps, "graph": True,
            "latency_us_per_batch": ms_max * 1e3 / (reps * n_graph),
            "value": edges_all / (ms_max / 1e3), "unit": UNIT, "gpu_launches_per_batch": launches,
            "note": "per-batch calls (batch-sized grids, under one wave) replayed as a CUDA graph: "
                    "launch-latency bound; the headline value is epoch mode"}


def e2e(args, tgl, sampler, chunks, mine, cfg, dev, world, full_d2h=False, gather_factory=None, events=None,
        cdev=None, batch_edges=None):
    """End to end through the public API with host buffers, copies inside the timed region.

    Per step: pinned host inputs -> H2D (copy stream) -> tgl_sample (compute stream) -> D2H of the
    step's result.  Inputs: with `batch_edges` (per chunk (e0, src, dst, neg, ts) of C.batch_edges) the
    mini-batch in TGL's own form -- the positive edges and their negatives, 16 bytes per 3 roots --
    expanded into roots on the device by tgl_batch_roots (R#16); else the root arrays themselves
    (8 bytes per root).  full_d2h=False: the result read back is the step's metric, the per-block
    (n_roots, nnz) counts (the blocks stay on the GPU for the consumer, as in TGL's training step);
    full_d2h=True: every block (offsets + nbr/eid/dt trimmed to nnz) is copied to pinned host memory.
    Double-buffered: the H2D of step j+1 and the D2H of step j overlap the sampling of j+1 / j+1.
    """
    L, S = len(cfg.fanouts), cfg.n_snapshots
    pinned = {}  # one pinned copy per distinct chunk (the step list cycles over them)
    for j, (r, t) in enumerate(chunks):
        if id(r) not in pinned:
            pinned[id(r)] = tuple(x.cpu().pin_memory() for x in batch_edges[j][1:]) if batch_edges is not None else \
                (r.cpu().pin_memory(), t.cpu().pin_memory())
    host = [pinned[id(r)] for r, _ in chunks]
    d_edges = None
    if batch_edges is not None:
        cap_e = max(x[1].numel() for x in batch_edges)
        d_edges = [tuple(torch.empty(cap_e, dtype=x.dtype, device=dev) for x in batch_edges[0][1:])
                   for _ in range(2)]
    host_ev = None
    if events is not None:  # step-6 events travel with their roots
        pin_ev = {k: (a.cpu().pin_memory(), b.cpu().pin_memory()) for k, (a, b) in events.items()}
        host_ev = [pin_ev[id(r)] for r, _ in chunks]
    cap_r = chunks[0][0].numel()
    d_ev = [(torch.empty(cap_r, dtype=torch.int32, device=dev), torch.empty(cap_r, dtype=torch.float32, device=dev))
            for _ in range(2)] if events is not None else None
    nb = L * S
    smps = [sampler, tgl.Sampler(sampler.g, cap_r, cfg.fanouts, cfg.strategy, S, cfg.snapshot_len,
                                 fused_gather=getattr(sampler, "_fused_spec", None) if sampler.fused_outs else None)]
    gathers = [gather_factory(smp) for smp in smps] if gather_factory is not None else None
    d_roots = [(torch.empty(cap_r, dtype=torch.int32, device=dev), torch.empty(cap_r, dtype=torch.float32, device=dev))
               for _ in range(2)]
    cnt_h = [torch.empty(2 * nb, dtype=torch.int64).pin_memory() for _ in range(2)]
    hb = None
    if full_d2h:
        hb = [[dict(off=torch.empty(b.offsets.numel(), dtype=torch.int64).pin_memory(),
                    nbr=torch.empty(b.nbr.numel(), dtype=torch.int32).pin_memory(),
                    eid=torch.empty(b.eid.numel(), dtype=torch.int32).pin_memory(),
                    dt=torch.empty(b.dt.numel(), dtype=torch.float32).pin_memory()) for b in smp.blocks]
              for smp in smps]
    comp = torch.cuda.current_stream()
    copy_s = torch.cuda.Stream()
    stats = dict(h2d=0, d2h=0, edges=0)
    roots_free = [None, None]  # compute finished reading d_roots[slot]
    outs_free = [None, None]   # copy stream finished reading smps[slot]'s blocks

    def run(js):
        pending = None  # (slot, event) whose counts / payload are still to be read
        for j in js:
            slot = j % 2
            dr, dt_ = d_roots[slot]
            n_r = chunks[j][0].numel()
            with torch.cuda.stream(copy_s):
                if roots_free[slot] is not None:
                    copy_s.wait_event(roots_free[slot])
                if d_edges is not None:  # the batch's edges + negatives
                    for dst_, src_ in zip(d_edges[slot], host[j]):
                        dst_[:src_.numel()].copy_(src_, non_blocking=True)
                    stats["h2d"] += sum(x.numel() * x.element_size() for x in host[j])
                else:
                    dr.copy_(host[j][0], non_blocking=True)
                    dt_.copy_(host[j][1], non_blocking=True)
                    stats["h2d"] += n_r * 8
                if host_ev is not None:
                    ne = host_ev[j][0].numel()
                    d_ev[slot][0][:ne].copy_(host_ev[j][0], non_blocking=True)
                    d_ev[slot][1][:ne].copy_(host_ev[j][1], non_blocking=True)
                    stats["h2d"] += ne * 8
                h2d_done = torch.cuda.Event()
                h2d_done.record(copy_s)
            comp.wait_event(h2d_done)
            if outs_free[slot] is not None:
                comp.wait_event(outs_free[slot])
            if d_edges is not None:
                tgl.batch_roots(*d_edges[slot], first_root=mine[j], n_roots=n_r, out=(dr, dt_))
            blocks = smps[slot].run(dr[:n_r], dt_[:n_r], seed=cfg.sampler_seed, root_key_base=mine[j])
            if gathers is not None:
                ev = None
                if host_ev is not None:
                    ne = host_ev[j][0].numel()
                    ev = (d_ev[slot][0][:ne], d_ev[slot][1][:ne])
                gathers[slot](dr, blocks[0], ev)
            for q, b in enumerate(blocks):
                cnt_h[slot][2 * q:2 * q + 1].copy_(b.n_roots_dev, non_blocking=True)
                cnt_h[slot][2 * q + 1:2 * q + 2].copy_(b.nnz_dev, non_blocking=True)
            done = torch.cuda.Event()
            done.record(comp)
            roots_free[slot] = done
            stats["d2h"] += 16 * nb
            if pending is not None:
                finish(*pending)
            pending = (slot, done)
        if pending is not None:
            finish(*pending)

    def finish(slot, done):
        done.synchronize()  # this step's counts are on the host
        c = cnt_h[slot]
        stats["edges"] += int(sum(int(c[2 * q + 1]) for q in range(nb)))
        if full_d2h:
            with torch.cuda.stream(copy_s):
                copy_s.wait_event(done)
                for q, b in enumerate(smps[slot].blocks):
                    n, z = int(c[2 * q]), int(c[2 * q + 1])
                    hb[slot][q]["off"][: n + 1].copy_(b.offsets[: n + 1], non_blocking=True)
                    hb[slot][q]["nbr"][:z].copy_(b.nbr[:z], non_blocking=True)
                    hb[slot][q]["eid"][:z].copy_(b.eid[:z], non_blocking=True)
                    hb[slot][q]["dt"][:z].copy_(b.dt[:z], non_blocking=True)
                    stats["d2h"] += (n + 1) * 8 + z * 12
                ev = torch.cuda.Event()
                ev.record(copy_s)
                outs_free[slot] = ev

    run(range(args.warmup))
    torch.cuda.synchronize(dev)
    stats.update(h2d=0, d2h=0, edges=0)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(comp)
    run(range(args.warmup, args.warmup + args.steps))
    comp.wait_stream(copy_s)
    e.record(comp)
    torch.cuda.synchronize(dev)
    ms = s.elapsed_time(e)
    edges, _, ms_max = reduce_report(stats["edges"], 0.0, ms, world, cdev or dev)
    src_what = ("pinned host mini-batch (positive edges src, dst, ts + negatives: 16 B per 3 roots) -> H2D -> "
                "tgl_batch_roots" if batch_edges is not None else "pinned host roots -> H2D")
    what = (f"{src_what} -> tgl_sample -> D2H of every block (offsets, nbr, eid, dt)" if full_d2h else
            f"{src_what} -> tgl_sample -> D2H of the step's metric (per-block n_roots, nnz); "
            "blocks stay on the GPU for the consumer")
    return {"value": edges / (ms_max / 1e3), "unit": UNIT, "h2d_bytes_per_step": stats["h2d"] // args.steps,
            "d2h_bytes_per_step": stats["d2h"] // args.steps,
            "kind": "full_d2h" if full_d2h else "device_consumer",
            "note": what + "; copy and compute streams overlapped"
                    + ("" if full_d2h else "; the blocks' own D2H is measured separately as e2e_full_d2h (PCIe-bound)")}


def parity_gate(args, cfg, tgl, sampler, src, dst, ts, chunks, mine, digests_by_start, rerun_same, world,
                want_cpu):
    """Parity of the TIMED configuration: the oracle samples whole timed chunks
    (every batch of a timed tgl_sample call, its key base = the batch's global root index); then
      * element by element: the first timed chunk re-run through the timed Sampler (same call, same
        launch configuration: 8.19 M roots = 32,000 tiles on C5) against the oracle's batches,
        concatenated (epoch mode == per-batch mode, R#7);
      * per-batch FNV-1a digests (tgl_block_digest) of every timed batch against the oracle's, on
        --parity-chunks distinct timed chunks (the digests of the other timed batches are reported
        for reproducibility; the last timed step's digests taken straight from the timed call's
        buffers must equal its re-run's).
    Also returns the CPU baseline (oracle as it stands, one thread, bounded sample; N = 1)."""
    B = cfg.batch
    L, S = len(cfg.fanouts), cfg.n_snapshots
    n_thr = max(1, host_info()["cores_available"] // max(1, world))
    timed = [mine[args.warmup + j] for j in range(args.steps)]
    distinct = list(dict.fromkeys(timed))
    # every rank checks its own chunks on the shared host: one chunk each at N > 1 (host RAM / cores)
    n_chk = max(1, min(args.parity_chunks if world == 1 else 1, len(distinct)))
    pick = [distinct[(len(distinct) - 1) * c // max(1, n_chk - 1)] if n_chk > 1 else distinct[0] for c in range(n_chk)]
    pick = list(dict.fromkeys(pick))
    by_start = {s0: chunks[args.warmup + timed.index(s0)] for s0 in pick}
    go, build_s = oracle_graph(cfg, src, dst, ts, [by_start[s0][0] for s0 in pick])
    ok_digest, checked_batches, first_mismatch, elem = True, 0, None, None
    cpu = None
    for idx, s0 in enumerate(pick):
        r, t = by_start[s0]
        r_np, t_np = r.cpu().numpy(), t.cpu().numpy()
        per_batch, secs = oracle_batches(go, cfg, r_np, t_np, s0, n_thr)
        od = oracle_batch_digests(per_batch, L * S)
        gd = digests_by_start[s0]
        same = od.shape == gd.shape and bool(np.array_equal(od, gd))
        if not same and first_mismatch is None:
            bad = np.argwhere(od != gd) if od.shape == gd.shape else [[-1, -1]]
            first_mismatch = f"chunk {s0}: block {int(bad[0][0])} batch {int(bad[0][1])}"
        ok_digest &= same
        checked_batches += gd.shape[1]
        if idx == 0:
            blocks = sampler.run(r, t, seed=cfg.sampler_seed, root_key_base=s0)  # the timed call
            ok, msg = compare_blocks(blocks, concat_batches(per_batch, L * S))
            n_edges = int(sum(len(bl[q]["nbr"]) for bl in per_batch for q in range(L * S)))
            elem = {"roots": int(r.numel()), "tiles_per_call": (int(r.numel()) + 255) // 256, "edges": n_edges,
                    "bit_exact": ok, "first_mismatch": msg}
            if want_cpu:
                cpu = cpu_baseline(args, cfg, go, build_s, r_np, t_np, s0,
                                   {"value": n_edges / secs, "unit": UNIT, "cores": n_thr, "seconds": secs,
                                    "sample": f"the whole chunk ({len(per_batch)} batches)"})
    n_timed_batches = sum((chunks[args.warmup + j][0].numel() + B - 1) // B for j in range(args.steps))
    bit_exact = bool(elem["bit_exact"] and ok_digest and rerun_same)
    return ({"bit_exact": bit_exact, "against": "oracle/ (CPU) on the timed chunks",
             "checked_roots": elem["roots"], "elementwise": elem,
             "digests": {"timed_batches": n_timed_batches,
                         "blocks_per_batch": L * S, "oracle_checked_batches": checked_batches,
                         "oracle_checked_chunks": len(pick), "match": ok_digest, "first_mismatch": first_mismatch,
                         "timed_call_equals_rerun": rerun_same,
                         "algorithm": "FNV-1a-64 per (batch, block): rebased int64 offsets, nbr, eid, dt bits "
                                      "(tgl_block_digest vs oracle.block_digest)"},
             "oracle_build_s": build_s}, cpu)


def cpu_baseline(args, cfg, go, build_s, r_np, t_np, key0, threaded):
    """Oracle as it stands, ONE thread on the host, on a bounded sample (consecutive batches of the
    first timed chunk, about --cpu-seconds of work), plus the same oracle over all host cores
    (threaded) on the whole chunk -- the parity run above."""
    B = cfg.batch
    nb_all = len(r_np) // B
    pilot = min(8, nb_all)
    _, secs = oracle_batches(go, cfg, r_np, t_np, key0, 1, n_batches=pilot)
    want = int(min(nb_all, max(pilot, args.cpu_seconds / max(secs / max(pilot, 1), 1e-6))))
    outs, secs = oracle_batches(go, cfg, r_np, t_np, key0, 1, n_batches=want)
    edges = sum(len(b["nbr"]) for bl in outs for b in bl)
    return {"value": edges / secs, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{want} consecutive batches x {B} roots ({want * B:,} roots, {edges:,} sampled edges) of the "
                      f"first timed chunk, single-threaded C oracle (-O2 -ffp-contract=off) on its T-CSR restricted "
                      f"to the chunk's nodes" + (" (sampler only: the oracle's gather / state write are not timed)"
                                                  if cfg.tables else ""),
            "seconds": secs, "oracle_x_threads": threaded, "oracle_tcsr_build_s": build_s, "host": host_info()}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    key = args.config
    cfg = C.CONFIGS[key]
    B = cfg.batch
    src, dst, ts, _ = setup_graph(key, cfg, dev)
    per_step = args.ref_batches
    n_chunks = args.warmup + args.steps
    starts = chunk_starts(cfg.n_roots_epoch, per_step * B, n_chunks, B)
    batches, bases = [], []
    for s0 in starts:
        r, t = C.roots(cfg, src, dst, ts, s0, per_step * B)
        for i in range(per_step):
            batches.append((r[i * B:(i + 1) * B], t[i * B:(i + 1) * B]))
            bases.append(s0 + i * B)
    w = args.warmup * per_step
    import oracle
    nodes = torch.cat([r for r, _ in batches])
    if len(cfg.fanouts) > 1:  # deeper layers' roots are sampled neighbours: every list may be read
        nodes = torch.arange(cfg.n_nodes, dtype=torch.int32, device=src.device)
    s_np, d_np, t_np, e_np, keep = C.relevant_substream(src, dst, ts, nodes, cfg.n_nodes, cfg.add_reverse)
    go = oracle.build_restricted(lambda: iter([(s_np, d_np, t_np, e_np, 0)]), n_nodes=cfg.n_nodes,
                                 add_reverse=cfg.add_reverse, keep=keep)
    strat = 0 if cfg.strategy == "most_recent" else 1
    host = [(r.cpu().numpy(), t.cpu().numpy()) for r, t in batches]
    edges, secs = 0, 0.0
    for q, ((r, t), base) in enumerate(zip(host, bases)):
        t0 = time.perf_counter()
        blocks = oracle.sample(go, r, t, fanouts=cfg.fanouts, strategy=strat, n_snapshots=cfg.n_snapshots,
                               snapshot_len=cfg.snapshot_len, seed=cfg.sampler_seed, root_key_base=base)
        dtm = time.perf_counter() - t0
        if q >= w:
            secs += dtm
            edges += sum(len(b["nbr"]) for b in blocks)
    value = edges / secs
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": secs * 1e3 / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
           "config": {"workload": workload_name(key, cfg), "batch_roots": B, "batches_per_step": per_step},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": f"{args.steps} steps x {per_step} batches x {B} roots, spread over the epoch"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def relaunch(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-run this command under torch.distributed.run with N
    local ranks (one process per GPU, rendezvous on 127.0.0.1), as the driver's N > 1 launch does."""
    import socket
    import subprocess
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_dry(args):
    """Host logic of the N-rank launch without a GPU (gloo): world size, the rank's chunk starts and
    the max-over-ranks / sum-of-work reduction, printed by rank 0 (tests/test_bench_host.py)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    cfg = C.CONFIGS[args.config]
    mine = rank_chunks(cfg.n_roots_epoch, args.batches * cfg.batch, args.steps, world, rank, cfg.batch)
    gathered = [None] * world
    if world > 1:
        dist.all_gather_object(gathered, mine)
    else:
        gathered = [mine]
    edges, _, ms = reduce_report(1000.0 * (rank + 1), 0.0, 2.0 + rank, world, torch.device("cpu"))
    if rank == 0:
        print(json.dumps({"n_gpus": world, "chunks": gathered, "edges": edges, "ms": ms}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="GPUs (ranks) of this node; outside torchrun N > 1 re-launches under torch.distributed.run")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=sorted(C.CONFIGS))
    ap.add_argument("--batches", type=int, default=0,
                    help="mini-batches per step (epoch mode); default 2048 for C5, 256 otherwise")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-batches", type=int, default=16, help="reference arm: batches per step")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--parity-chunks", type=int, default=2,
                    help="distinct timed chunks whose per-batch digests are checked against the oracle")
    ap.add_argument("--distinct", type=int, default=32, help="distinct root chunks (cycled over the steps)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-per-batch", action="store_true")
    ap.add_argument("--sharding", default="root", choices=["root", "node"],
                    help="root: replicated T-CSR, roots sharded (default); node: node-sharded T-CSR (SURVEY 8(e))")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--separate-gather", action="store_true",
                    help="configs with tables (C3): gather the sampled edges' rows with separate tgl_gather launches "
                         "instead of the copy kernel's fused gather (tgl_fused_gather, default)")
    ap.add_argument("--dry-run", action="store_true", help=argparse.SUPPRESS)  # host logic only (gloo, no GPU)
    args = ap.parse_args()
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and (args.gpus or 1) > 1:
        sys.exit(relaunch(args.gpus))
    world = int(world_env or 1)
    if args.gpus is None:
        args.gpus = world
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.batches <= 0:
        args.batches = 2048 if args.config == "C5" else 256
    if args.dry_run:
        return run_dry(args)
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_node_sharded(args) if args.sharding == "node" else run_ours(args)


if __name__ == "__main__":
    main()
