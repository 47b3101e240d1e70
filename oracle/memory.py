"""Closed-form memory model: Eq. 1 and Eq. 2.

Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations


def eq1_elements(entries: int, horizon: int, nodes: int, features: int) -> int:
    """Eq. 1: size = 2[(entries - (2 horizon - 1)) x horizon x nodes x features]
    elements after Alg. 1 (x and y stacks, T_in = T_out = horizon)."""
    return 2 * ((entries - (2 * horizon - 1)) * horizon * nodes * features)


def materialized_elements(E: int, T_in: int, T_out: int, N: int, F: int) -> int:
    """Eq. 1 generalised to T_in != T_out: S windows of T_in + T_out slices
    each, S = E - T_in - T_out + 1 (reading c11).  Equals eq1_elements when
    T_in = T_out = horizon."""
    S = E - T_in - T_out + 1
    return S * (T_in + T_out) * N * F


def eq2_elements(entries: int, horizon: int, nodes: int, features: int) -> tuple[int, int]:
    """Eq. 2: index_batching_size = entries x nodes x features
    + (entries - (2 horizon - 1)).  Returned as (data elements, index entries)
    because the paper adds quantities of different widths (reading c12)."""
    return entries * nodes * features, entries - (2 * horizon - 1)


def index_elements(E: int, T_in: int, T_out: int, N: int, F: int) -> tuple[int, int]:
    """Eq. 2 generalised: one copy of the data plus one start index per window."""
    return E * N * F, E - T_in - T_out + 1


def index_bytes(E, T_in, T_out, N, F, elem_bytes=4, idx_bytes=8) -> int:
    """Eq. 2 in bytes: data elements at their width plus index entries counted as 8-byte
    integers (reading c12); idx_bytes=4 gives the device footprint of the int32
    plan libpgti keeps."""
    d, i = index_elements(E, T_in, T_out, N, F)
    return d * elem_bytes + i * idx_bytes


def ratio(E, T_in, T_out, N, F, elem_bytes=8, idx_bytes=8) -> float:
    """Materialised / index-batched bytes (Eq. 1 / Eq. 2, reading c12; 8-byte index entries,
    S:281 -- idx_bytes=4 for the int32 device plan)."""
    return materialized_elements(E, T_in, T_out, N, F) * elem_bytes / \
        index_bytes(E, T_in, T_out, N, F, elem_bytes, idx_bytes)


def halo_shard_rows(S_r: int, T_in: int, T_out: int) -> int:
    """Rows a rank holds under halo sharding: its S_r window starts plus the
    T_in + T_out - 1 rows the last window reaches past them (BASELINE.json
    north_star)."""
    return S_r + T_in + T_out - 1
