"""CPU checks of the C ABI: the library builds, loads and exports every symbol include/pgti.h
declares; host-only entry points (pgti_graph_build) agree with the oracle; host shard logic."""
import os
import re

import numpy as np
import pytest

import synth
from oracle import philox, transitions, windows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="session")
def pgti():
    from paper_2507_11683_b200 import build
    build.build()
    from paper_2507_11683_b200 import pgti as mod
    return mod


def test_exports_every_declared_symbol(pgti):
    import ctypes
    hdr = open(os.path.join(ROOT, "include", "pgti.h")).read()
    declared = set(re.findall(r"\b(pgti_[a-z0-9_]+)\s*\(", hdr))
    assert len(declared) >= 20
    lib = ctypes.CDLL(pgti.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert pgti.version().startswith("libpgti")


def test_sm100a_cubin_and_no_fallback(pgti):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pgti.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out, out


@pytest.mark.parametrize("N,p,seed", [(7, 0.4, 1), (30, 0.1, 2), (1, 1.0, 3)])
def test_graph_build_matches_oracle(pgti, N, p, seed):
    src, dst, w = synth.random_graph(N, p, seed)
    csr = pgti.graph_build(N, src, dst, w)
    Pf, Pb = transitions.transition_matrices(N, src, dst, w, dense=True)

    def dense(rowptr, col, val):
        D = np.zeros((N, N))
        for i in range(N):
            for e in range(rowptr[i], rowptr[i + 1]):
                D[i, col[e]] = val[e]
            assert np.all(np.diff(col[rowptr[i]:rowptr[i + 1]]) > 0)  # ascending columns
        return D

    tol = dict(rtol=1e-7, atol=0)
    assert np.allclose(dense(csr["a_rowptr"], csr["a_col"], csr["Pf_val"]), Pf, **tol)
    assert np.allclose(dense(csr["a_rowptr"], csr["a_col"], csr["PbT_val"]), Pb.T, **tol)
    assert np.allclose(dense(csr["at_rowptr"], csr["at_col"], csr["Pb_val"]), Pb, **tol)
    assert np.allclose(dense(csr["at_rowptr"], csr["at_col"], csr["PfT_val"]), Pf.T, **tol)


def test_graph_build_errors(pgti):
    with pytest.raises(pgti.PgtiError) as e:
        pgti.graph_build(3, [0, 0], [1, 1], [1.0, 2.0])
    assert e.value.name == "INVALID_ARG" and "duplicate" in str(e.value)
    with pytest.raises(pgti.PgtiError):
        pgti.graph_build(3, [0], [5], [1.0])
    with pytest.raises(pgti.PgtiError):
        pgti.graph_build(3, [0], [1], [-1.0])


@pytest.mark.parametrize("N,rows,graph", [(207, 16, "knn"), (37, 7, "er"), (100, 1, "knn"),
                                           (45, 64, "ring"), (2716, 32, "knn")])
def test_graph_windows_plan(pgti, N, rows, graph):
    """SpMM staging plan (pgti_graph_windows): each window's list is exactly the sorted set of
    its rows' columns and lcol maps every CSR entry back to its column (brute force)."""
    g = {"er": lambda: synth.random_graph(N, 0.15, seed=N), "knn": lambda: synth.make_graph(N, 8),
         "ring": lambda: synth.ring_graph(N)}[graph]()
    csr = pgti.graph_build(N, *g)
    full = pgti.add_windows(csr, N, rows)
    mx = 0
    for pat in ("a", "at"):
        rp, col = csr[pat + "_rowptr"], csr[pat + "_col"]
        wp, wn = full[pat + "_win_ptr"], full[pat + "_win_nodes"]
        lc = full[pat + "_lcol"].view(np.uint16)
        nwin = -(-N // rows)
        assert wp.shape == (nwin + 1,) and wp[0] == 0
        for w in range(nwin):
            r0, r1 = w * rows, min(N, (w + 1) * rows)
            u = wn[wp[w]:wp[w + 1]]
            assert np.array_equal(u, np.unique(col[rp[r0]:rp[r1]]))
            e = np.arange(rp[r0], rp[r1])
            assert np.array_equal(u[lc[e]], col[e])
            mx = max(mx, u.size)
    assert full["win_max"] == mx and full["win_rows"] == rows
    assert pgti.add_windows(csr, N, 0)["win_rows"] == 0


def test_graph_windows_errors(pgti):
    csr = pgti.graph_build(4, [0, 1], [1, 2], [1.0, 1.0])
    for rows in (0, 65):
        with pytest.raises(pgti.PgtiError) as e:
            pgti.graph_windows(4, csr["a_rowptr"], csr["a_col"], rows)
        assert e.value.name == "INVALID_ARG"
    bad = csr["a_col"].copy()
    bad[0] = 9
    with pytest.raises(pgti.PgtiError):
        pgti.graph_windows(4, csr["a_rowptr"], bad, 2)


def test_desc_mirror_matches_the_library(pgti):
    import ctypes
    assert pgti._desc_size == ctypes.sizeof(pgti.DcrnnDesc)
    assert pgti.DcrnnDesc.cheb.offset + 4 <= ctypes.sizeof(pgti.DcrnnDesc)


def test_desc_validation_without_gpu(pgti):
    m = pgti.DCRNN(207, 2, 1, 2, 64, 2, 12, 12, 64, 416, None)
    with pytest.raises(pgti.PgtiError):  # K > 0 needs CSR pointers
        m.num_params()
    m = pgti.DCRNN(207, 2, 1, 2, 64, 0, 12, 12, 64, 416, None)
    assert m.num_params() == 2 * 0 + synth.num_params(synth.CONFIGS["metr_la"].replace(K=0))
    bad = pgti.DCRNN(207, 2, 1, 2, 64, 0, 12, 13, 64, 416, None)  # T_out > T_in
    with pytest.raises(pgti.PgtiError):
        bad.workspace_bytes()


@pytest.mark.parametrize("name", list(synth.CONFIGS))
def test_shard_plan_vs_oracle(pgti, name):
    from paper_2507_11683_b200 import trainer
    cfg = synth.CONFIGS[name]
    S = windows.num_windows(cfg.E, cfg.T_in, cfg.T_out)
    assert trainer.window_count(cfg.E, cfg.T_in, cfg.T_out) == S
    S_tr = windows.split_counts(S)[0]
    assert trainer.train_windows(S) == S_tr
    assert trainer.val_windows(S) == windows.split_counts(S)[1]
    for R in (1, 2, 4, 8):
        covered = []
        for r in range(R):
            p = trainer.shard_plan(S_tr, R, r, cfg.T_in, cfg.T_out)
            a, S_r = philox.shard(S_tr, R, r)
            assert (p.win_lo, p.win_hi) == (a, a + S_r)
            r0, r1 = philox.shard_rows(S_tr, R, r, cfg.T_in, cfg.T_out)
            assert p.row_lo == r0 and p.row_hi >= r1 and p.row_hi <= cfg.E
            assert p.row_lo <= p.stat_lo <= p.stat_hi <= p.row_hi
            covered.append((p.stat_lo, p.stat_hi))
        # the statistics row ranges tile every row a training window reads
        assert covered[0][0] == 0 and covered[-1][1] == S_tr + cfg.T_in - 1
        assert all(covered[i][1] == covered[i + 1][0] for i in range(R - 1))
    assert trainer.row_pitch(207, 2) == 416 and trainer.row_pitch(325, 2) == 652


@pytest.mark.parametrize("E,N,F,T_in,T_out,seed", [(60, 12, 2, 3, 2, 0), (521, 20, 1, 4, 1, 1),
                                                   (200, 7, 3, 12, 12, 2)])
def test_stats_finalize_matches_alg1(pgti, E, N, F, T_in, T_out, seed):
    """pgti_stats_finalize (host part of pgti_series_moments) turns the three sums over the
    STACKED x_train (Alg. 1, here formed literally by the oracle) into Alg. 1's
    mean and population std (lines 201-202) to 1e-12, about shift 0 and about the mean."""
    rng = np.random.default_rng(seed)
    v = (50.0 + 10.0 * rng.standard_normal((E, N, F))).astype(np.float32)
    x, _ = windows.alg1_stack(v.astype(np.float64), T_in, T_out)
    x_train = x[:windows.split_counts(x.shape[0])[0]]
    mu_ref, sd_ref = windows.alg1_stats(v, T_in, T_out)
    for shift in (0.0, mu_ref, -3.25):
        d = x_train - shift
        mean, var = pgti.stats_finalize((d.size, d.sum(), (d * d).sum()), shift)
        assert abs(mean - mu_ref) <= 1e-12 * abs(mu_ref), (shift, mean, mu_ref)
        # about shift 0 the one-pass form E[v^2] - E[v]^2 cancels ~ (mu/sigma)^2 = 25 -> 2.5e-14 rel
        assert abs(np.sqrt(var) - sd_ref) <= 1e-12 * sd_ref, (shift, np.sqrt(var), sd_ref)


def test_stats_finalize_errors(pgti):
    with pytest.raises(pgti.PgtiError) as e:
        pgti.stats_finalize((0.0, 0.0, 0.0), 0.0)
    assert e.value.name == "TOO_FEW_ENTRIES"
    with pytest.raises(pgti.PgtiError) as e:
        pgti.stats_finalize((4.0, float("nan"), 1.0), 0.0)
    assert e.value.name == "NONFINITE"
    # values {1, 2}: mean 1.5, var 0.25; a constant series has var 0 (clamped, never < 0)
    assert pgti.stats_finalize((2.0, 3.0, 5.0), 0.0) == (1.5, 0.25)
    assert pgti.stats_finalize((3.0, 6.0, 12.0), 0.0) == (2.0, 0.0)
