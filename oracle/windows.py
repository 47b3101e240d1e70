"""Alg. 1 written out literally, in float64 where it computes.

Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np


def num_windows(E: int, T_in: int, T_out: int) -> int:
    """Number of (x, y) snapshot pairs: every placement of a T_in-step input
    window followed by its T_out-step target inside E entries.

    P:297 prints "entries - 2 x horizon - 1" and Eq. 2 prints
    "entries - (2 x horizon - 1)"; Fig. 3 (E=6, horizon 3 -> exactly one
    snapshot, x = G0..G2, y = G3..G5) fixes the second reading, generalised to
    T_in != T_out (reading c11): S = E - T_in - T_out + 1.
    """
    return max(0, E - T_in - T_out + 1)


def split_counts(S: int) -> tuple[int, int, int]:
    """70/10/20 train/val/test split over windows (Alg. 1:
    x_train = x[:round(len(x) * 0.70)]).  Python's round(), as Alg. 1 is Python
    (reading c10: no ties occur at the configs)."""
    n_train = round(S * 0.70)
    n_test = round(S * 0.20)
    return n_train, S - n_train - n_test, n_test


def alg1_stack(v: np.ndarray, T_in: int, T_out: int, starts=None):
    """Alg. 1: for each window, x.append(data[window]),
    y.append(data[window + horizon]); then stack.  ``starts`` restricts the
    loop to a subset of windows (the same definition on fewer windows, used
    when the full stack would not fit in host RAM -- the paper's OOM).

    Returns (x[S][T_in][N][F], y[S][T_out][N][F]) with v's dtype.
    """
    S = num_windows(v.shape[0], T_in, T_out)
    if starts is None:
        starts = range(S)
    x, y = [], []
    for s in starts:
        s = int(s)
        assert 0 <= s < S, f"window start {s} outside [0, {S})"
        x.append(v[s:s + T_in])
        y.append(v[s + T_in:s + T_in + T_out])
    return np.stack(x, axis=0), np.stack(y, axis=0)


def alg1_stats(v: np.ndarray, T_in: int, T_out: int) -> tuple[float, float]:
    """Alg. 1 lines 199-202 literally: stack every x snapshot (float64), take
    x_train = x[:round(len(x)*0.70)], mu = mean(x_train), sigma = std(x_train)
    (population std; scalar over all nodes and features -- reading c9)."""
    x, _ = alg1_stack(v.astype(np.float64), T_in, T_out)
    n_train = split_counts(x.shape[0])[0]
    x_train = x[:n_train]
    return float(np.mean(x_train)), float(np.std(x_train))


def standardize32(a: np.ndarray, mu: float, sigma: float) -> np.ndarray:
    """Alg. 1, (a - mu) / sigma, evaluated in IEEE float32:
    fl32(fl32(a - fl32(mu)) / fl32(sigma)) (reading O4: the series is stored in
    float32; mu, sigma computed in float64 and applied rounded to float32)."""
    a32 = np.asarray(a, dtype=np.float32)
    return ((a32 - np.float32(mu)) / np.float32(sigma)).astype(np.float32)


def materialize(v: np.ndarray, T_in: int, T_out: int, mu: float, sigma: float, starts=None):
    """The standard PGT/Alg. 1 pipeline: stack every snapshot, then
    standardise x and y with the training statistics (the
    StaticGraphTemporalSignal lists of P:180).  Returns float32 arrays
    features[S][T_in][N][F], targets[S][T_out][N][F]."""
    x, y = alg1_stack(v, T_in, T_out, starts)
    return standardize32(x, mu, sigma), standardize32(y, mu, sigma)
