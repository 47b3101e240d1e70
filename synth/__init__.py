"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no windows, statistics,
normalisation, transition matrices, diffusion, GRU, loss or optimiser).  It
only draws the raw inputs the method consumes, with the shapes of the paper's
workloads (Table 1; BASELINE.json configs), following the
recipe written down in DESIGN.md "Input recipe":

* ``CONFIGS``          -- the five workload shapes (CP, ML, PB, PAL, PE).
* ``make_graph``       -- directed kNN sensor graph as an edge list (src, dst,
                          w) with self loops; weights are a thresholded
                          Gaussian kernel of distance ("a simple
                          transformation ... weighted matrix").
* ``make_series``      -- raw float32 series ``v[E][N][F]`` (any row range
                          can be generated independently, for halo shards).
* ``make_params``      -- flat float32 parameter vector (uniform init).

Seeds: data 0, graph 1, params 2, shuffle 3.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED_DATA, SEED_GRAPH, SEED_PARAMS, SEED_SHUFFLE = 0, 1, 2, 3


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    N: int          # sensors (graph nodes)
    E: int          # time entries in the series
    F: int          # features per node
    T_in: int
    T_out: int
    L: int          # stacked DCGRU layers
    H: int          # hidden units
    K: int          # diffusion hops (M = 2K+1 blocks)
    B: int          # per-GPU batch
    F_out: int = 1  # predicted channels (channel 0)
    knn: int = 8    # out-neighbours per node before thresholding
    period: int = 288  # samples per day (5-min data) / 52 weeks for CP
    cheb: bool = False  # diffusion blocks by the Chebyshev recurrence (Li et al.'s code, c25)

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


# BASELINE.json "configs"; SURVEY.md section 8 config table.
CONFIGS = {
    "chickenpox": Config("chickenpox", N=20, E=521, F=1, T_in=4, T_out=1, L=1, H=32, K=2,
                         B=4, knn=4, period=52),
    "metr_la": Config("metr_la", N=207, E=34272, F=2, T_in=12, T_out=12, L=2, H=64, K=2, B=64),
    "pems_bay": Config("pems_bay", N=325, E=52116, F=2, T_in=12, T_out=12, L=2, H=64, K=2, B=64),
    "pems_all_la": Config("pems_all_la", N=2716, E=105120, F=2, T_in=12, T_out=12, L=2, H=64,
                          K=2, B=64),
    "pems": Config("pems", N=11160, E=105120, F=2, T_in=12, T_out=12, L=2, H=64, K=2, B=64),
}


# --------------------------------------------------------------------------- graph
def _hilbert_index(x: np.ndarray, y: np.ndarray, order: int = 16) -> np.ndarray:
    """Position along a Hilbert curve of integer points (locality ordering)."""
    n = 1 << order
    x = x.astype(np.int64).copy()
    y = y.astype(np.int64).copy()
    d = np.zeros_like(x)
    s = n // 2
    while s > 0:
        rx = ((x & s) > 0).astype(np.int64)
        ry = ((y & s) > 0).astype(np.int64)
        d += s * s * ((3 * rx) ^ ry)
        flip = (ry == 0) & (rx == 1)
        x = np.where(flip, n - 1 - x, x)
        y = np.where(flip, n - 1 - y, y)
        swap = ry == 0
        x, y = np.where(swap, y, x), np.where(swap, x, y)
        s //= 2
    return d


def make_graph(N: int, knn: int = 8, seed: int = SEED_GRAPH, kappa: float = 0.1):
    """Directed kNN graph on N random points in the unit square.

    Nodes are numbered in Hilbert-curve order.  Node i gets an edge i->j to
    each of its ``knn`` nearest neighbours with weight exp(-(d/s)^2), s = the
    median of all kNN distances (gives ~8.3 nnz/row at knn=8, matching METR-LA's
    1,722/207 [ext]); weights below ``kappa`` are dropped
    (Li et al.'s normalized_k threshold) and a self loop of weight 1 is added.
    Weights are float32 values (both sides read the same numbers).

    Returns (src int32[nnz], dst int32[nnz], w float32[nnz]) sorted by (src, dst).
    """
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(seed)
    pts = rng.random((N, 2))
    q = np.minimum((pts * 65536).astype(np.int64), 65535)
    order = np.argsort(_hilbert_index(q[:, 0], q[:, 1]), kind="stable")
    pts = pts[order]
    k = min(knn, N - 1)
    src, dst, w = [np.arange(N)], [np.arange(N)], [np.ones(N)]
    if k > 0:
        dist, nbr = cKDTree(pts).query(pts, k=k + 1)
        dist, nbr = dist[:, 1:], nbr[:, 1:]
        s = float(np.percentile(dist, 50)) or 1.0
        wk = np.exp(-(dist / s) ** 2)
        keep = (wk >= kappa) & (nbr != np.arange(N)[:, None])
        rows = np.repeat(np.arange(N), k).reshape(N, k)
        src.append(rows[keep])
        dst.append(nbr[keep])
        w.append(wk[keep])
    src = np.concatenate(src).astype(np.int32)
    dst = np.concatenate(dst).astype(np.int32)
    w = np.concatenate(w).astype(np.float32)
    o = np.lexsort((dst, src))
    src, dst, w = src[o], dst[o], w[o]
    dup = (np.diff(src) == 0) & (np.diff(dst) == 0)
    if dup.any():
        keep = np.concatenate([[True], ~dup])
        src, dst, w = src[keep], dst[keep], w[keep]
    return src, dst, w


def ring_graph(N: int, weight: float = 1.0, self_loops: bool = False):
    """Directed ring i -> (i+1) mod N (test graphs)."""
    src = np.arange(N, dtype=np.int32)
    dst = ((np.arange(N) + 1) % N).astype(np.int32)
    w = np.full(N, weight, dtype=np.float32)
    if self_loops:
        src = np.concatenate([src, np.arange(N, dtype=np.int32)])
        dst = np.concatenate([dst, np.arange(N, dtype=np.int32)])
        w = np.concatenate([w, np.ones(N, np.float32)])
    o = np.lexsort((dst, src))
    return src[o], dst[o], w[o]


def random_graph(N: int, p: float, seed: int, self_loops: bool = True):
    """Erdos-Renyi directed graph with random float32 weights in [0.1, 1] (tests)."""
    rng = np.random.default_rng(seed)
    mask = rng.random((N, N)) < p
    if self_loops:
        np.fill_diagonal(mask, True)
    src, dst = np.nonzero(mask)
    w = (0.1 + 0.9 * rng.random(src.size)).astype(np.float32)
    return src.astype(np.int32), dst.astype(np.int32), w


# --------------------------------------------------------------------------- series
_CHUNK = 4096
_BURN = 96


def _noise_chunk(N: int, c: int, seed: int, rows: int, nbr_mix) -> np.ndarray:
    """Spatially mixed AR(1) noise for time chunk c, float64 [rows][N].

    Each chunk is drawn from its own stream (seed, c) with a burn-in, so any
    row range can be generated without generating its predecessors.
    """
    rng = np.random.default_rng([seed, c])
    xi = rng.standard_normal((_BURN + rows, N))
    from scipy.signal import lfilter

    e = lfilter([0.436], [1.0, -0.9], xi, axis=0)[_BURN:]
    if nbr_mix is not None:
        e = 0.5 * e + 0.5 * np.asarray(nbr_mix @ e.T).T
    return e


def _neighbour_mean(N: int, knn: int, seed: int):
    """Unweighted mean over each node's kNN list (data-generating process only)."""
    import scipy.sparse as sp

    src, dst, _ = make_graph(N, knn, seed)
    cnt = np.bincount(src, minlength=N).astype(np.float64)
    return sp.csr_matrix((1.0 / cnt[src], (src, dst)), shape=(N, N))


def make_series(cfg: Config, seed: int = SEED_DATA, row_lo: int = 0, row_hi: int | None = None,
                graph_seed: int = SEED_GRAPH) -> np.ndarray:
    """Raw series rows [row_lo, row_hi) of v[E][N][F] as float32 (finite, sigma > 0).

    Traffic shapes (F=2): channel 0 "speed" = 55 + 10 sin(2 pi (t mod 288)/288 + phi_n)
    + 4 e[t, n], e a graph-coupled AR(1); channel 1 = time of day (t mod 288)/288
    (SURVEY reading c8).  Chickenpox shape (F=1): non-negative integer counts with a
    52-week season.
    """
    row_hi = cfg.E if row_hi is None else row_hi
    assert 0 <= row_lo <= row_hi <= cfg.E
    N, F = cfg.N, cfg.F
    out = np.empty((row_hi - row_lo, N, F), np.float32)
    phi = np.random.default_rng([seed, 1 << 20]).random(N) * 2 * math.pi
    mix = _neighbour_mean(N, cfg.knn, graph_seed) if N > 1 else None
    c0, c1 = row_lo // _CHUNK, (row_hi - 1) // _CHUNK if row_hi > row_lo else -1
    for c in range(c0, c1 + 1):
        t0 = c * _CHUNK
        rows = min(_CHUNK, cfg.E - t0)
        e = _noise_chunk(N, c, seed, rows, mix)
        t = np.arange(t0, t0 + rows)
        a, b = max(row_lo, t0), min(row_hi, t0 + rows)
        sl = slice(a - t0, b - t0)
        season = 2 * math.pi * (t[sl] % cfg.period) / cfg.period
        if F == 1:
            lam = 20 + 10 * np.sin(season[:, None] + phi[None, :]) + 5 * e[sl]
            out[a - row_lo:b - row_lo, :, 0] = np.round(np.maximum(lam, 0.0))
        else:
            out[a - row_lo:b - row_lo, :, 0] = 55 + 10 * np.sin(season[:, None] + phi[None, :]) \
                + 4 * e[sl]
            out[a - row_lo:b - row_lo, :, 1] = ((t[sl] % cfg.period) / cfg.period)[:, None]
            for f in range(2, F):
                out[a - row_lo:b - row_lo, :, f] = e[sl] * 0.5
    return out


# --------------------------------------------------------------------------- params
def param_shapes(cfg: Config, model: str = "stepwise"):
    """Parameter blocks in flat order; model "encdec": the encoder
    layers, then the decoder layers (layer-0 input F_out channels), then the readout."""
    M = 2 * cfg.K + 1
    shapes = []
    stacks = [("", cfg.F)] + ([("dec", cfg.F_out)] if model == "encdec" else [])
    for pre, f0 in stacks:
        for l in range(cfg.L):
            c_in = (f0 if l == 0 else cfg.H) + cfg.H
            shapes += [(f"W_ru{pre}{l}", (M, c_in, 2 * cfg.H)), (f"b_ru{pre}{l}", (2 * cfg.H,)),
                       (f"W_c{pre}{l}", (M, c_in, cfg.H)), (f"b_c{pre}{l}", (cfg.H,))]
    shapes += [("W_out", (cfg.H, cfg.F_out)), ("b_out", (cfg.F_out,))]
    return shapes


def num_params(cfg: Config, model: str = "stepwise") -> int:
    return sum(int(np.prod(s)) for _, s in param_shapes(cfg, model))


def make_params(cfg: Config, seed: int = SEED_PARAMS, kind: str = "random",
                scale: float = 1.0, model: str = "stepwise") -> np.ndarray:
    """Flat float32 parameters.  ``kind="random"``: every entry (biases too)
    uniform in +-scale/sqrt(fan_in), to exercise every path in parity tests;
    ``kind="train"``: weights as above, b_ru = 1, other biases 0 (Li et al.'s
    bias_start, [ext])."""
    rng = np.random.default_rng(seed)
    parts = []
    for name, shp in param_shapes(cfg, model):
        fan_in = shp[0] * shp[1] if len(shp) == 3 else (shp[0] if name == "W_out" else cfg.H)
        bound = scale / math.sqrt(fan_in)
        p = rng.uniform(-bound, bound, size=shp)
        if kind == "train" and name.startswith("b_"):
            p = np.full(shp, 1.0 if name.startswith("b_ru") else 0.0)
        parts.append(p.reshape(-1))
    return np.concatenate(parts).astype(np.float32)
