"""Philox4x32-10 and the per-epoch index plan (reading c16).

Philox4x32-10 is the counter-based generator of Salmon et al. (SC'11,
"Parallel random numbers: as easy as 1, 2, 3"; Random123), written out here
independently of the CUDA side, which implements the same generator.

Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np

_MASK = np.uint64(0xFFFFFFFF)
_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = np.uint64(0x9E3779B9), np.uint64(0xBB67AE85)


def philox4x32_10(ctr, key):
    """ctr: 4 arrays (or ints) of 32-bit words, key: 2 words.  Returns 4 uint64
    arrays holding the 32-bit output words.

    Round (Random123 philox4x32round): (hi0, lo0) = M0 * c0, (hi1, lo1) = M1 * c2,
    c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); key bumped by (W0, W1)
    before every round but the first; 10 rounds.
    """
    c = [np.asarray(w, dtype=np.uint64) & _MASK for w in ctr]
    k0, k1 = (np.asarray(w, dtype=np.uint64) & _MASK for w in key)
    for r in range(10):
        if r > 0:
            k0 = (k0 + _W0) & _MASK
            k1 = (k1 + _W1) & _MASK
        p0 = _M0 * c[0]
        p1 = _M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return c


def window_keys(seed: int, epoch: int, rank: int, n: int) -> np.ndarray:
    """Sort key of window i (0 <= i < n) for this (seed, epoch, rank):
    the first two output words of Philox4x32-10 with
    ctr = (i, epoch_lo, epoch_hi, rank), key = (seed_lo, seed_hi),
    as the u64 (w0 << 32) | w1 (reading O6)."""
    i = np.arange(n, dtype=np.uint64)
    e = np.uint64(epoch)
    s = np.uint64(seed)
    out = philox4x32_10((i, e & _MASK, e >> np.uint64(32), np.uint64(rank)),
                        (s & _MASK, s >> np.uint64(32)))
    return (out[0] << np.uint64(32)) | out[1]


def epoch_permutation(seed: int, epoch: int, rank: int, n: int) -> np.ndarray:
    """pi = argsort of (key_i, i): "the dataset is shuffled at the start of each
    epoch", the mechanism being unstated (reading c16)."""
    keys = window_keys(seed, epoch, rank, n)
    return np.lexsort((np.arange(n), keys)).astype(np.int64)


def shard(S_tr: int, R: int, r: int) -> tuple[int, int]:
    """Rank r's window range under halo sharding: starts [a_r, a_r + S_r),
    S_r = floor(S_tr / R), a_r = r S_r (the S_tr mod R remainder is dropped so
    every rank runs the same number of steps -- reading c17)."""
    S_r = S_tr // R
    return r * S_r, S_r


def index_plan(S_tr: int, R: int, r: int, B: int, seed: int, epoch: int,
               shuffle: bool = True) -> np.ndarray:
    """Global window starts rank r visits this epoch, in order: a_r + pi(i),
    truncated to floor(S_r/B) B (drop_last).  Batch j is entries
    [jB, (j+1)B)."""
    a_r, S_r = shard(S_tr, R, r)
    perm = epoch_permutation(seed, epoch, r, S_r) if shuffle else np.arange(S_r)
    n_used = (S_r // B) * B
    return (a_r + perm[:n_used]).astype(np.int64)


def shard_rows(S_tr: int, R: int, r: int, T_in: int, T_out: int) -> tuple[int, int]:
    """Global series rows [row0, row1) rank r must hold: the rows its windows
    read, i.e. S_r starts plus a halo of T_in + T_out - 1 rows."""
    a_r, S_r = shard(S_tr, R, r)
    return a_r, a_r + S_r + T_in + T_out - 1


def batch_plan(S_tr: int, R: int, r: int, B: int, seed: int, epoch: int) -> np.ndarray:
    """Generalized-distributed-index-batching's local shuffle (SURVEY A10/A11,
    NEXT f4): the partition (rank r's shard, as in `index_plan`) is fixed and so is every batch's
    MEMBERSHIP -- batch j holds the consecutive windows a_r + [jB, (j+1)B) -- while the ORDER of
    the floor(S_r/B) batches is shuffled each epoch by the same Philox key construction applied to
    batch indices (ctr = (j, epoch_lo, epoch_hi, r)).  Returns the window starts in visiting
    order (n_used = floor(S_r/B) B entries)."""
    a_r, S_r = shard(S_tr, R, r)
    nb = S_r // B
    order = epoch_permutation(seed, epoch, r, nb)
    return (a_r + (order[:, None] * B + np.arange(B)[None, :]).reshape(-1)).astype(np.int64)


def global_plan(S_tr: int, R: int, r: int, B: int, seed: int, epoch: int) -> np.ndarray:
    """Distributed-index-batching with replicated data and communication-free GLOBAL shuffling
    (SURVEY A6/A7, NEXT f1): every rank holds the whole series and derives the same
    permutation of all S_tr training windows (Philox ctr rank word fixed to 0); rank r visits
    slice [r S_r, (r+1) S_r) of it, truncated to whole batches.  The R slices are disjoint and
    together cover R S_r windows of the one global order."""
    S_r = S_tr // R
    perm = epoch_permutation(seed, epoch, 0, S_tr)
    mine = perm[r * S_r:(r + 1) * S_r]
    return mine[:(S_r // B) * B].astype(np.int64)
