"""Pins for oracle.windows / oracle.memory (Alg. 1, Eq. 1, Eq. 2, Table 1)."""
import csv
import math
import os

import numpy as np
import pytest

from oracle import memory, windows

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_window_count_bruteforce():
    # every (T_in, T_out) placement enumerated by hand
    for E in range(1, 30):
        for T_in in range(1, 6):
            for T_out in range(1, 6):
                starts = [s for s in range(E) if s + T_in + T_out <= E]
                assert windows.num_windows(E, T_in, T_out) == len(starts)


def test_fig3_worked_example():
    # P:302 / P:177: horizon 3 over G0..G5 -> one snapshot, x = G0..G2, y = G3..G5
    v = np.arange(6, dtype=np.float32).reshape(6, 1, 1)
    assert windows.num_windows(6, 3, 3) == 1
    x, y = windows.alg1_stack(v, 3, 3)
    assert x.shape == (1, 3, 1, 1) and y.shape == (1, 3, 1, 1)
    assert x.ravel().tolist() == [0, 1, 2] and y.ravel().tolist() == [3, 4, 5]


def test_window_counts_at_configs():
    # S:143 "E=105120, horizon=12 -> count = 105097"; METR-LA 34,249
    assert windows.num_windows(105120, 12, 12) == 105097
    assert windows.num_windows(34272, 12, 12) == 34249
    assert windows.num_windows(521, 4, 1) == 517


def test_split_counts():
    assert windows.split_counts(34249) == (23974, 3425, 6850)
    assert windows.split_counts(105097) == (73568, 10510, 21019)
    n_tr, n_va, n_te = windows.split_counts(517)
    assert (n_tr, n_tr + n_va + n_te) == (362, 517)


def test_spec_stats_example():
    # E=6, h=1, values 0..5 -> 5 windows, train = 4 -> mu 1.5, sigma sqrt(1.25)
    v = np.arange(6, dtype=np.float32).reshape(6, 1, 1)
    mu, sigma = windows.alg1_stats(v, 1, 1)
    assert mu == 1.5 and math.isclose(sigma, math.sqrt(1.25), rel_tol=1e-15)


@pytest.mark.parametrize("seed", range(5))
def test_stats_closed_form_weights(seed):
    # window-weighted closed form: row t is covered by
    # w(t) = min(t, S_tr-1) - max(0, t-T_in+1) + 1 training windows
    rng = np.random.default_rng(seed)
    E, N, F = int(rng.integers(20, 60)), int(rng.integers(1, 4)), int(rng.integers(1, 3))
    T_in, T_out = int(rng.integers(1, 6)), int(rng.integers(1, 6))
    v = rng.normal(3, 2, (E, N, F)).astype(np.float32)
    mu, sigma = windows.alg1_stats(v, T_in, T_out)
    S = windows.num_windows(E, T_in, T_out)
    S_tr = windows.split_counts(S)[0]
    t = np.arange(E)
    w = np.clip(np.minimum(t, S_tr - 1) - np.maximum(0, t - T_in + 1) + 1, 0, None)
    vv = v.astype(np.float64).reshape(E, -1)
    cnt = w.sum() * N * F
    mu2 = (w[:, None] * vv).sum() / cnt
    var2 = (w[:, None] * (vv - mu2) ** 2).sum() / cnt
    assert abs(mu2 - mu) <= 1e-12 * abs(mu)
    assert abs(math.sqrt(var2) - sigma) <= 1e-12 * sigma


def test_standardize_values():
    # [2, 4], mu 3, sigma 1 -> [-1, 1]; mu 0, sigma 1 -> unchanged
    assert windows.standardize32(np.array([2.0, 4.0]), 3.0, 1.0).tolist() == [-1.0, 1.0]
    a = np.random.default_rng(0).normal(size=100).astype(np.float32)
    assert np.array_equal(windows.standardize32(a, 0.0, 1.0), a)


def test_standardized_train_moments():
    # standardized training x has window-weighted mean ~0 and variance ~1
    rng = np.random.default_rng(7)
    v = rng.normal(50, 8, (80, 3, 2)).astype(np.float32)
    mu, sigma = windows.alg1_stats(v, 4, 3)
    x, _ = windows.materialize(v, 4, 3, mu, sigma)
    xt = x[:windows.split_counts(x.shape[0])[0]].astype(np.float64)
    assert abs(xt.mean()) < 1e-6 and abs(xt.std() - 1) < 1e-6  # float32 storage


def test_materialize_is_view_of_series():
    # every snapshot equals the standardised series slice (views == copies)
    rng = np.random.default_rng(3)
    v = rng.normal(size=(40, 5, 2)).astype(np.float32)
    mu, sigma = 0.1, 1.3
    x, y = windows.materialize(v, 5, 3, mu, sigma)
    z = windows.standardize32(v, mu, sigma)
    for s in range(x.shape[0]):
        assert np.array_equal(x[s], z[s:s + 5]) and np.array_equal(y[s], z[s + 5:s + 8])


def _unit(u):
    return {"KB": 1e3, "MB": 1e6, "GiB": 2 ** 30}[u]


def test_table1_eq1_reproduces_paper():
    with open(os.path.join(GOLD, "table1.csv")) as f:
        rows = list(csv.DictReader(r for r in f if not r.startswith("#")))
    assert len(rows) == 6
    for r in rows:
        E, N, F, h = (int(r[k]) for k in ("entries", "nodes", "features", "horizon"))
        size = memory.eq1_elements(E, h, N, F) * 8 / _unit(r["after_unit"])
        assert round(size, 2) == float(r["after_value"]), (r["dataset"], size)
        assert memory.materialized_elements(E, h, h, N, F) == memory.eq1_elements(E, h, N, F)


def test_eq1_equals_materialized_nbytes():
    # measured bytes of the Alg. 1 stacks equal Eq. 1 exactly
    rng = np.random.default_rng(1)
    for E, h, N, F in [(100, 4, 3, 2), (30, 3, 2, 1), (50, 7, 4, 3)]:
        v = rng.normal(size=(E, N, F))
        x, y = windows.alg1_stack(v, h, h)
        assert x.nbytes + y.nbytes == memory.eq1_elements(E, h, N, F) * 8
    assert memory.eq1_elements(100, 4, 3, 2) == 4464
    v = rng.normal(size=(60, 3, 2))
    x, y = windows.alg1_stack(v, 5, 2)
    assert x.size + y.size == memory.materialized_elements(60, 5, 2, 3, 2)


def test_eq2_and_ratio():
    d, i = memory.eq2_elements(105120, 12, 11160, 2)
    assert d == 105120 * 11160 * 2 and i == 105097
    assert memory.index_elements(105120, 12, 12, 11160, 2) == (d, i)
    # closed-form ratio ~24x at h=12 (-95.8 %)
    r = memory.ratio(105120, 12, 12, 11160, 2)
    assert 23.9 < r < 24.0 and abs((1 - 1 / r) - 0.958) < 1e-3
    # Chickenpox: Eq. 1 bytes 657,920 (Table 1) over 521*20*8 data + 514 8-byte indices
    assert memory.ratio(521, 4, 4, 20, 1) == 657920 / (83360 + 514 * 8)
    # the int32 device plan (idx_bytes=4)
    assert memory.ratio(521, 4, 4, 20, 1, idx_bytes=4) == 657920 / (83360 + 514 * 4)
    assert memory.index_bytes(521, 4, 4, 20, 1, elem_bytes=8) == 83360 + 514 * 8


def test_table1_before_sizes_are_eq2_data_term():
    # Table 1 "Size Before Preprocessing" = the single data copy that
    # index-batching keeps (Eq. 2's first term) at float64: 83.36 KB, 44.59 MB
    assert round(memory.index_elements(521, 4, 4, 20, 1)[0] * 8 / 1e3, 2) == 83.36
    assert round(memory.index_elements(17472, 8, 8, 319, 1)[0] * 8 / 1e6, 2) == 44.59


def test_halo_rows_bruteforce():
    from oracle import philox
    for S_tr in (10, 37, 362):
        for R in (1, 2, 4, 8):
            for r in range(R):
                T_in, T_out = 4, 3
                a, S_r = philox.shard(S_tr, R, r)
                rows = set()
                for s in range(a, a + S_r):
                    rows.update(range(s, s + T_in + T_out))
                r0, r1 = philox.shard_rows(S_tr, R, r, T_in, T_out)
                if S_r:
                    assert (min(rows), max(rows) + 1) == (r0, r1)
                    assert r1 - r0 == memory.halo_shard_rows(S_r, T_in, T_out)
