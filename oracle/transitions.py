"""Random-walk transition matrices of the diffusion convolution.

P_f = D_O^-1 A and P_b = D_I^-1 A^T (Li et al., ICLR'18, Eq. 2 [ext]); PAPER.md
P:222 states PGT-DCRNN "implements the diffusion convolution operations
described in" Li et al.; P:163 defines A as the weighted adjacency of the
static graph.  A[i][j] = weight of the directed edge i -> j.  A zero degree
gives a zero row (reading c5).

Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def adjacency(N: int, src, dst, w, dense: bool = False):
    """Weighted adjacency A (float64) from an edge list."""
    A = sp.csr_matrix((np.asarray(w, np.float64), (np.asarray(src), np.asarray(dst))),
                      shape=(N, N))
    return A.toarray() if dense else A


def transition_matrices(N: int, src, dst, w, dense: bool = False):
    """Returns (P_f, P_b) with D_O = diag(A 1), D_I = diag(A^T 1)."""
    A = adjacency(N, src, dst, w, dense=False)
    d_out = np.asarray(A.sum(axis=1)).ravel()
    d_in = np.asarray(A.sum(axis=0)).ravel()
    inv_out = np.where(d_out > 0, 1.0 / np.where(d_out > 0, d_out, 1.0), 0.0)
    inv_in = np.where(d_in > 0, 1.0 / np.where(d_in > 0, d_in, 1.0), 0.0)
    Pf = sp.diags(inv_out) @ A
    Pb = sp.diags(inv_in) @ A.T
    if dense:
        return Pf.toarray(), Pb.toarray()
    return sp.csr_matrix(Pf), sp.csr_matrix(Pb)
