"""Host logic of bench.py (no GPU): the algorithmic-bytes model, root-sharded chunk assignment,
and the max-over-ranks / sum-of-work reporting under torch.distributed (gloo, world_size 2)."""
import math
import os
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from synth import configs as C  # noqa: E402


def test_algorithmic_bytes_model_c5():
    cfg = C.CONFIGS["C5"]                      # 1 layer, S = 3, t_s = 5: 80 B / root + 24 B / edge
    assert bench.algorithmic_bytes(cfg, [1], [0]) == 80
    assert bench.algorithmic_bytes(cfg, [1000], [6300]) == 80 * 1000 + 24 * 6300


def test_algorithmic_bytes_model_two_layer():
    cfg = C.CONFIGS["C2"]                      # L = 2, S = 1, t_s = inf
    # layer 0: 8 + 16 + 8 + 8 = 40 / root, 28 / edge; layer 1: 8 + 16 + 8 + 8 = 40 / root, 24 / edge
    assert bench.algorithmic_bytes(cfg, [600, 6000], [6000, 60000]) == 40 * 600 + 28 * 6000 + 40 * 6000 + 24 * 60000


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_rank_chunks_disjoint_cover(world):
    cfg = C.CONFIGS["C5"]
    chunk, steps = 2048 * cfg.batch, 33
    per_rank = [bench.rank_chunks(cfg.n_roots_epoch, chunk, steps, world, r, cfg.batch) for r in range(world)]
    allc = sorted(x for p in per_rank for x in p)
    assert len(set(allc)) == len(allc) == steps * world               # disjoint
    assert all(x % cfg.batch == 0 for x in allc)                       # batch aligned
    assert all(0 <= x <= cfg.n_roots_epoch - chunk for x in allc)
    gaps = [b - a for a, b in zip(allc, allc[1:])]
    assert min(gaps) >= chunk                                          # chunks never overlap


REPORT = textwrap.dedent(r'''
    import os, sys
    sys.path.insert(0, os.environ["REPO"])
    import torch, torch.distributed as dist
    import bench
    dist.init_process_group("gloo")
    r = dist.get_rank()
    e, b, ms = bench.reduce_report(100.0 * (r + 1), 10.0, 5.0 + r, 2, torch.device("cpu"))
    assert (e, b, ms) == (300.0, 20.0, 6.0), (e, b, ms)
    print("ok", r)
    dist.destroy_process_group()
''')


def test_reduce_report_gloo_world2(tmp_path):
    script = tmp_path / "rep.py"
    script.write_text(REPORT)
    env = dict(os.environ, REPO=ROOT)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(script)],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    assert r.stdout.count("ok") == 2


def test_workload_names_distinct_and_shared_by_both_arms():
    """One config.workload per config, used by our arm, the node-sharded mode and the reference arm."""
    names = {k: bench.workload_name(k, C.CONFIGS[k]) for k in C.CONFIGS}
    assert len(set(names.values())) == len(names)
    assert names["C5"].startswith("C5 ") and "121,000,000 nodes" in names["C5"] and "3 snapshot(s) of 5" in names["C5"]
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert src.count('"workload": workload_name(key, cfg)') == 3


@pytest.mark.parametrize("n", [2])
def test_gpus_flag_self_launches_n_ranks(n):
    """`bench.py --gpus N` outside torchrun re-launches itself with N ranks (gloo here, --dry-run:
    host logic only) -- n_gpus in the line is the real world size and the ranks' chunks are disjoint."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "4",
                        "--dry-run"], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    import json
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == n
    starts = [s for rank_chunks in line["chunks"] for s in rank_chunks]
    assert len(starts) == 4 * n and len(set(starts)) == len(starts)
    assert line["edges"] == sum(1000.0 * (q + 1) for q in range(n)) and line["ms"] == 2.0 + n - 1


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
