"""Pins for oracle.philox: Random123 known answers, permutation semantics."""
import itertools
import os

import numpy as np

from oracle import philox

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_known_answer_vectors():
    rows = [l.split() for l in open(os.path.join(GOLD, "philox_kat.txt")) if not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        w = [int(h, 16) for h in r]
        out = philox.philox4x32_10(w[0:4], w[4:6])
        assert [int(o) for o in out] == w[6:10], r


def test_permutation_is_permutation_and_deterministic():
    for n in (1, 2, 17, 1000):
        p = philox.epoch_permutation(3, 5, 0, n)
        assert sorted(p.tolist()) == list(range(n))
        assert np.array_equal(p, philox.epoch_permutation(3, 5, 0, n))
    assert not np.array_equal(philox.epoch_permutation(3, 5, 0, 100),
                              philox.epoch_permutation(3, 6, 0, 100))


def test_keys_vectorised_equals_scalar():
    keys = philox.window_keys(0x123456789, 7, 3, 10)
    for i in range(10):
        o = philox.philox4x32_10([i, 7, 0, 3], [0x23456789, 0x1])
        assert int(keys[i]) == (int(o[0]) << 32) | int(o[1])


def test_chi2_uniform_permutations():
    # over 10,000 epochs at count 4 every one of the 24 orders appears 1/24 +- 3 sigma
    counts = {p: 0 for p in itertools.permutations(range(4))}
    n = 10000
    for e in range(n):
        counts[tuple(philox.epoch_permutation(11, e, 0, 4).tolist())] += 1
    p = 1 / 24
    sd = (n * p * (1 - p)) ** 0.5
    assert all(abs(c - n * p) < 4 * sd for c in counts.values()), counts


def test_index_plan_shards():
    S_tr, B = 103, 4
    for R in (1, 2, 4, 8):
        seen = []
        for r in range(R):
            plan = philox.index_plan(S_tr, R, r, B, seed=3, epoch=2)
            a, S_r = philox.shard(S_tr, R, r)
            assert len(plan) == (S_r // B) * B
            assert plan.min() >= a and plan.max() < a + S_r
            assert len(set(plan.tolist())) == len(plan)
            seen += plan.tolist()
        assert len(set(seen)) == len(seen)
    ident = philox.index_plan(S_tr, 1, 0, B, 3, 2, shuffle=False)
    assert ident.tolist() == list(range(100))
