"""Dev tool: write the row-normalised kNN transition CSR of a workload's synthetic sensor graph
as int32 N, int32 nnz, int32 rowptr[N+1], int32 col[nnz], float32 val[nnz] (spmm_tiled_mb.cu)."""
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, __file__.rsplit("/tests/", 1)[0])
from synth import CONFIGS, make_graph  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
src, dst, w = make_graph(cfg.N, knn=cfg.knn)
A = sp.csr_matrix((w, (src, dst)), shape=(cfg.N, cfg.N))
A.sum_duplicates()
A.sort_indices()
d = np.asarray(A.sum(axis=1)).ravel()
P = sp.diags(1.0 / d) @ A
P = P.tocsr()
P.sort_indices()
with open(sys.argv[2], "wb") as f:
    np.array([cfg.N, P.nnz], np.int32).tofile(f)
    P.indptr.astype(np.int32).tofile(f)
    P.indices.astype(np.int32).tofile(f)
    P.data.astype(np.float32).tofile(f)
print(cfg.N, P.nnz)
