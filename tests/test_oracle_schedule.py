"""Pins for Alg. 2 random chunk scheduling in the oracle (reading R#26), no GPU:
the start offset is a multiple of cs below bs, uniform over epochs (chi-square); batches are
consecutive, disjoint, bs long, and stop exactly when the next would pass |E|; cs = bs gives the
plain schedule starting at 0 (Alg. 1's training loop)."""
import numpy as np

import oracle


def test_schedule_structure():
    for n, bs, cs in [(10_000, 600, 100), (599, 600, 100), (600, 600, 600), (157_474, 600, 60), (0, 8, 2)]:
        for epoch in range(20):
            st = oracle.chunk_schedule(n, bs, cs, epoch, seed=42)
            if not st:  # not even one batch fits after the random start
                assert n < 2 * bs
                continue
            e_s = st[0]
            assert e_s % cs == 0 and 0 <= e_s < bs
            assert all(b - a == bs for a, b in zip(st, st[1:]))
            assert st[-1] + bs <= n < st[-1] + 2 * bs
    assert all(oracle.chunk_schedule(10_000, 600, 600, e, seed=7)[0] == 0 for e in range(10))


def test_start_uniform_over_epochs():
    from scipy.stats import chisquare
    bs, cs = 4000, 250
    starts = [oracle.chunk_schedule(1_000_000, bs, cs, e, seed=123)[0] // cs for e in range(16_000)]
    counts = np.bincount(starts, minlength=bs // cs)
    assert len(counts) == bs // cs
    assert chisquare(counts).pvalue > 1e-4
