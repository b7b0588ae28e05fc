"""Small run of every libtgl.so kernel family for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): T-CSR build (full and node range), sampler (most_recent S = 3 with finite
windows, uniform 2-layer, the validity / dedup / replacement / root-time variants, > 64 tiles so the
super / hyper tile bases run), gather, state write, digest, chunk schedule, node-sharded sampling
and node state over 2 in-process ranks.  Results are compared with the oracle where cheap; the
point of the run is the sanitizer's report (scripts/sanitize.sh).

python tools/sanitize_run.py
"""
import math
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: expected values)
import paper_2203_14883_b200 as tgl  # noqa: E402
from synth.tiny import random_graph, random_roots  # noqa: E402


def main():
    small = os.environ.get("SANITIZE_SMALL") == "1"  # racecheck: fewer tiles (it is slow)
    V, E = (800, 12000) if small else (3000, 60000)
    src, dst, ts, eid = random_graph(11, V, E, with_eid=True, integer_times=True)
    s, d, t, e = (torch.as_tensor(x).cuda() for x in (src, dst, ts, eid))
    g = tgl.build(s, d, t, e, n_nodes=V, add_reverse=True)
    go = oracle.build(src, dst, ts, eid, n_nodes=V, add_reverse=True)
    assert np.array_equal(g.indptr.cpu().numpy(), go["indptr"])
    roots, rts = random_roots(5, V, 20_000 if small else 70_000)   # 274 tiles: super tile bases
    r, rt = torch.as_tensor(roots).cuda(), torch.as_tensor(rts).cuda()
    for fan, strat, S, tsl, kw in (([10], "most_recent", 3, 5.0, {}), ([10, 5], "uniform", 1, math.inf, {}),
                                   ([4, 3], "uniform", 2, 20.0, {}), ([6], "uniform", 1, math.inf, {"replacement": True}),
                                   ([5, 5], "most_recent", 1, math.inf, {"hop_time": "root", "dedup": True})):
        blocks = tgl.sample(g, r, rt, fanouts=fan, strategy=strat, n_snapshots=S, snapshot_len=tsl, seed=3,
                            root_key_base=100, **kw)
        bo = oracle.sample(go, roots, rts, fanouts=fan, strategy=0 if strat == "most_recent" else 1, n_snapshots=S,
                           snapshot_len=tsl, seed=3, root_key_base=100, **kw)
        for b, o in zip(blocks, bo):
            off, nbr, _, dt, _ = b.trimmed()
            assert np.array_equal(off.cpu().numpy(), o["offsets"]) and np.array_equal(nbr.cpu().numpy(), o["nbr"])
        bounds = torch.tensor(list(range(0, r.numel() + 1, 5000)), dtype=torch.int64, device="cuda")
        tgl.block_digest(blocks[0], bounds)
    assert g.codec["n_codes"] > 0  # integer times 0..50: the time codec (codes, packed records) runs
    # a graph with real-valued times: no codec, 16-byte slot records
    src2, dst2, ts2, _ = random_graph(12, V, E, integer_times=False)
    g2 = tgl.build(*(torch.as_tensor(x).cuda() for x in (src2, dst2, ts2)), n_nodes=V, add_reverse=True)
    assert g2.codec["n_codes"] == 0
    go2 = oracle.build(src2, dst2, ts2, n_nodes=V, add_reverse=True)
    roots2, rts2 = random_roots(6, V, 20_000 if small else 70_000, integer_times=False)
    for fan, strat, S, tsl in (([10], "most_recent", 3, 5.0), ([6, 4], "uniform", 1, math.inf)):
        blocks = tgl.sample(g2, torch.as_tensor(roots2).cuda(), torch.as_tensor(rts2).cuda(), fanouts=fan,
                            strategy=strat, n_snapshots=S, snapshot_len=tsl, seed=5)
        bo = oracle.sample(go2, roots2, rts2, fanouts=fan, strategy=0 if strat == "most_recent" else 1, n_snapshots=S,
                           snapshot_len=tsl, seed=5)
        for b, o in zip(blocks, bo):
            assert np.array_equal(b.trimmed()[1].cpu().numpy(), o["nbr"])
    valid = torch.full(((E + 31) // 32,), -1, dtype=torch.int32, device="cuda")
    tgl.edge_valid_set(valid, torch.arange(0, E, 3, dtype=torch.int32, device="cuda"), False, n_bits=E)
    for strat in ("most_recent", "uniform"):
        tgl.sample(g, r[:5000], rt[:5000], fanouts=[5, 3], strategy=strat, seed=1, edge_valid=valid)
    table = torch.randn(V, 33, device="cuda")
    out = tgl.gather(r[:4000], [table])[0]
    assert torch.equal(out, table[r[:4000].long()])
    ring = torch.zeros(V * 3, 9, device="cuda")
    pos = torch.zeros(V, dtype=torch.int32, device="cuda")
    tgl.state_write(r[:5000], rt[:5000], [(torch.randn(5000, 9, device="cuda"), ring)], n_nodes=V, K=3, pos=pos)
    tgl.chunk_schedule(E, 600, 100, 2, 7)
    # node-sharded: 2 ranks on threads
    W = 2
    indptr = tgl.tcsr_indptr(s, d, t, n_nodes=V, add_reverse=True)
    from paper_2203_14883_b200.sharded import edge_balanced_splits
    sp = [int(x) for x in edge_balanced_splits(indptr, W).cpu()]
    shards = [tgl.build_range(s, d, t, e, n_nodes=V, add_reverse=True, node_lo=sp[q], node_hi=sp[q + 1],
                              n_local_stored=int(indptr[sp[q + 1]] - indptr[sp[q]])) for q in range(W)]
    grp = tgl.ShardGroup(W)
    smps = [tgl.ShardSampler(shards[q], sp, q, W, 4000, [5, 4], "uniform", 2, 20.0, group=grp) for q in range(W)]
    mem = [torch.randn(sp[q + 1] - sp[q], 8, device="cuda") for q in range(W)]
    errs = []

    def work(q):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                smps[q].run(r[q * 4000:(q + 1) * 4000], rt[q * 4000:(q + 1) * 4000], seed=3, root_key_base=q * 4000)
                smps[q].gather(r[:3000], [mem[q]])
                smps[q].state_write(r[:3000], rt[:3000], [(torch.randn(3000, 8, device="cuda"), mem[q])])
                st.synchronize()
        except Exception as ex:  # noqa: BLE001
            errs.append(ex)
    th = [threading.Thread(target=work, args=(q,)) for q in range(W)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    assert tgl.check(g) == 0 and tgl.check(None) == 0
    torch.cuda.synchronize()
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
