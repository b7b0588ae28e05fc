"""Small random temporal graphs for parity tests (numpy, seeded).

Inputs only: chronological edge streams with deliberate ties, self-loops, isolated
nodes and hubs, plus root lists with duplicated nodes at different times
and out-of-window times.  No method arithmetic.
"""
from __future__ import annotations

import numpy as np


def random_graph(seed: int, n_nodes: int, n_edges: int, *, t_max: float = 50.0,
                 integer_times: bool = True, hub_frac: float = 0.3, with_eid: bool = False):
    rng = np.random.default_rng(seed)
    n_nodes = max(int(n_nodes), 1)
    # skewed endpoints: a few hubs take hub_frac of the edges
    hubs = rng.integers(0, n_nodes, size=max(1, n_nodes // 8))
    pick_hub = rng.random(n_edges) < hub_frac
    src = np.where(pick_hub, rng.choice(hubs, size=n_edges), rng.integers(0, n_nodes, size=n_edges))
    dst = rng.integers(0, n_nodes, size=n_edges)
    if integer_times:
        ts = np.sort(rng.integers(0, int(t_max) + 1, size=n_edges)).astype(np.float32)   # many ties
    else:
        ts = np.sort(rng.random(n_edges) * t_max).astype(np.float32)
    eid = rng.permutation(n_edges).astype(np.int32) if with_eid else None
    return src.astype(np.int32), dst.astype(np.int32), ts, eid


def random_roots(seed: int, n_nodes: int, n_roots: int, *, t_max: float = 50.0,
                 integer_times: bool = True):
    rng = np.random.default_rng(seed + 7919)
    nodes = rng.integers(0, max(n_nodes, 1), size=n_roots)
    if n_roots >= 4:                       # duplicated roots at different timestamps
        nodes[1::4] = nodes[0::4][: len(nodes[1::4])]
    if integer_times:
        t = rng.integers(0, int(t_max) + 3, size=n_roots).astype(np.float32)
    else:
        t = (rng.random(n_roots) * (t_max + 2)).astype(np.float32)
    return nodes.astype(np.int32), t
