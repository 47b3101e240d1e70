"""Pins for oracle.philox: Random123 known answers, permutation semantics."""
import itertools
import os

import numpy as np
import pytest

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


@pytest.mark.parametrize("S_tr,R,B", [(1000, 1, 8), (1000, 4, 16), (37, 2, 5)])
def test_batch_plan_membership_frozen_order_shuffled(S_tr, R, B):
    """f4: each batch is a consecutive block of the rank's shard, the blocks are a
    permutation of the shard's whole batches, and the order changes between epochs."""
    orders = []
    for r in range(R):
        a_r, S_r = philox.shard(S_tr, R, r)
        nb = S_r // B
        for epoch in (0, 1):
            p = philox.batch_plan(S_tr, R, r, B, 3, epoch)
            assert p.size == nb * B
            blocks = p.reshape(nb, B)
            assert np.all(np.diff(blocks, axis=1) == 1)          # membership: consecutive
            starts = (blocks[:, 0] - a_r) // B
            assert np.all((blocks[:, 0] - a_r) % B == 0)
            assert sorted(starts.tolist()) == list(range(nb))   # every whole batch once
            orders.append(tuple(starts))
    if S_tr // R // B > 3:
        assert orders[0] != orders[1]
    assert np.array_equal(philox.batch_plan(S_tr, R, 0, B, 3, 1),
                          philox.batch_plan(S_tr, R, 0, B, 3, 1))


@pytest.mark.parametrize("S_tr,R,B", [(1000, 1, 8), (1000, 4, 16), (1003, 8, 4)])
def test_global_plan_slices_one_permutation(S_tr, R, B):
    """f1: the ranks' slices are disjoint, each lies in [0, S_tr), and their
    concatenation (before batch truncation) is a prefix of one global permutation that every
    rank derives identically (no exchange)."""
    S_r = S_tr // R
    seen = []
    for r in range(R):
        p = philox.global_plan(S_tr, R, r, B, 3, 2)
        assert p.size == (S_r // B) * B and p.min() >= 0 and p.max() < S_tr
        seen.append(p)
    allw = np.concatenate(seen)
    assert np.unique(allw).size == allw.size
    perm = philox.epoch_permutation(3, 2, 0, S_tr)
    for r in range(R):
        assert np.array_equal(seen[r], perm[r * S_r:r * S_r + (S_r // B) * B])
    # a global shuffle mixes the time axis across ranks (unlike the halo shard)
    if R > 1:
        assert seen[0].max() >= S_r
