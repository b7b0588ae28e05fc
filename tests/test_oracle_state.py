"""Pins for the oracle's state write (Fig. 2 step 6; reading R#25), no GPU:
  * K = 1 (node memory): each touched node holds the row of its LAST event (numpy: last
    occurrence via np.unique on the reversed ids); untouched rows are unchanged;
  * K > 1 (mailbox ring): after the batch, node v's ring read from its cursor backwards holds the
    K most recent of (its previous ring contents ++ its new events) -- a history model built
    with numpy, not the sequential ring loop;
  * cursor arithmetic: pos[v] advances by the number of v's events mod K;
  * out-of-range ids are skipped and reported.
"""
import numpy as np
import pytest

import oracle


def test_k1_last_event_wins():
    rng = np.random.default_rng(0)
    V, n, w = 50, 400, 7
    ids = rng.integers(0, V, n).astype(np.int32)
    ts = np.sort(rng.random(n).astype(np.float32))
    rows = rng.standard_normal((n, w)).astype(np.float32)
    table = rng.standard_normal((V, w)).astype(np.float32)
    before = table.copy()
    tts = np.full(V, -1.0, np.float32)
    assert oracle.state_write(ids, ts, n_nodes=V, K=1, tables=[(rows, table)], ts_table=tts) == 0
    u, last_rev = np.unique(ids[::-1], return_index=True)
    last = n - 1 - last_rev
    np.testing.assert_array_equal(table[u], rows[last])
    np.testing.assert_array_equal(tts[u], ts[last])
    untouched = np.setdiff1d(np.arange(V), u)
    np.testing.assert_array_equal(table[untouched], before[untouched])


@pytest.mark.parametrize("K", [2, 3, 10])
def test_ring_holds_k_most_recent(K):
    rng = np.random.default_rng(K)
    V, w = 30, 3
    table = np.zeros((V * K, w), np.float32)
    tts = np.zeros(V * K, np.float32)
    pos = rng.integers(0, K, V).astype(np.int32)
    # history model: per node, the list of all rows ever written, oldest first
    hist = {v: [] for v in range(V)}
    # seed rings with a first batch so old contents matter
    for batch in range(3):
        n = int(rng.integers(1, 120))
        ids = (rng.zipf(1.5, n) % V).astype(np.int32)
        ts = (batch * 1000 + np.sort(rng.integers(0, 1000, n))).astype(np.float32)
        rows = rng.standard_normal((n, w)).astype(np.float32)
        pos_before = pos.copy()
        assert oracle.state_write(ids, ts, n_nodes=V, K=K, tables=[(rows, table)], pos=pos, ts_table=tts) == 0
        for i in range(n):
            hist[int(ids[i])].append((rows[i], ts[i]))
        counts = np.bincount(ids, minlength=V)
        np.testing.assert_array_equal(pos, (pos_before + counts) % K)
        for v in range(V):
            recent = hist[v][-K:]
            # slot of the j-th most recent (j = 1..len): (pos[v] - j) mod K
            for j, (r, t) in enumerate(reversed(recent), start=1):
                slot = v * K + (int(pos[v]) - j) % K
                np.testing.assert_array_equal(table[slot], r)
                assert tts[slot] == t


def test_out_of_range_ids_skipped():
    ids = np.array([0, 5, -1, 2], np.int32)
    rows = np.arange(8, dtype=np.float32).reshape(4, 2)
    table = np.zeros((3, 2), np.float32)
    assert oracle.state_write(ids, np.zeros(4, np.float32), n_nodes=3, K=1, tables=[(rows, table)]) == -2
    np.testing.assert_array_equal(table, [[0, 1], [0, 0], [6, 7]])


def test_several_tables_share_cursors():
    rng = np.random.default_rng(5)
    V, K, n = 9, 4, 60
    ids = rng.integers(0, V, n).astype(np.int32)
    a_rows, b_rows = rng.standard_normal((n, 5)).astype(np.float32), rng.integers(0, 9, (n, 2)).astype(np.int64)
    a1, b1 = np.zeros((V * K, 5), np.float32), np.zeros((V * K, 2), np.int64)
    a2, b2 = a1.copy(), b1.copy()
    p1, p2, p3 = [np.arange(V, dtype=np.int32) % K for _ in range(3)]
    oracle.state_write(ids, np.zeros(n, np.float32), n_nodes=V, K=K, tables=[(a_rows, a1), (b_rows, b1)], pos=p1)
    oracle.state_write(ids, np.zeros(n, np.float32), n_nodes=V, K=K, tables=[(a_rows, a2)], pos=p2)
    oracle.state_write(ids, np.zeros(n, np.float32), n_nodes=V, K=K, tables=[(b_rows, b2)], pos=p3)
    np.testing.assert_array_equal(a1, a2)
    np.testing.assert_array_equal(b1, b2)
    np.testing.assert_array_equal(p1, p2)
