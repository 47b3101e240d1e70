// Host-side transition-matrix construction on the two CSR patterns (pgti_graph_build).
// P_f = D_O^-1 A, P_b = D_I^-1 A^T (Li et al. Eq. 2 [ext]; PAPER.md P:163, P:222;
// DESIGN.md readings c1, c4, c5).  Degrees are summed in double; values stored as float.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "common.cuh"

extern "C" pgti_status pgti_graph_build(int32_t N, int64_t nnz, const int32_t *src,
                                        const int32_t *dst, const float *w, int32_t *a_rowptr,
                                        int32_t *a_col, float *Pf_val, float *PbT_val,
                                        int32_t *at_rowptr, int32_t *at_col, float *Pb_val,
                                        float *PfT_val) {
  pgti::clear_error();
  PGTI_REQUIRE(N > 0 && nnz >= 0, PGTI_ERR_INVALID_ARG, "pgti_graph_build: N=%d nnz=%lld", N,
               (long long)nnz);
  PGTI_REQUIRE(nnz < (int64_t(1) << 31), PGTI_ERR_INVALID_ARG, "nnz %lld exceeds int32",
               (long long)nnz);
  PGTI_REQUIRE((nnz == 0 || (src && dst && w)) && a_rowptr && at_rowptr &&
                   (nnz == 0 || (a_col && Pf_val && PbT_val && at_col && Pb_val && PfT_val)),
               PGTI_ERR_INVALID_ARG, "pgti_graph_build: null pointer");
  std::vector<double> d_out(N, 0.0), d_in(N, 0.0);
  for (int64_t e = 0; e < nnz; ++e) {
    PGTI_REQUIRE(src[e] >= 0 && src[e] < N && dst[e] >= 0 && dst[e] < N, PGTI_ERR_INVALID_ARG,
                 "edge %lld (%d -> %d) outside [0, %d)", (long long)e, src[e], dst[e], N);
    PGTI_REQUIRE(std::isfinite(w[e]) && w[e] >= 0.f, PGTI_ERR_INVALID_ARG,
                 "edge %lld has weight %g (must be finite, >= 0)", (long long)e, (double)w[e]);
    d_out[src[e]] += w[e];
    d_in[dst[e]] += w[e];
  }
  auto inv = [](double d) { return d > 0.0 ? 1.0 / d : 0.0; };

  // pattern(A): order edges by (src, dst)
  std::vector<int64_t> ord(nnz);
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
    return src[a] != src[b] ? src[a] < src[b] : dst[a] < dst[b];
  });
  for (int64_t i = 1; i < nnz; ++i)
    PGTI_REQUIRE(!(src[ord[i]] == src[ord[i - 1]] && dst[ord[i]] == dst[ord[i - 1]]),
                 PGTI_ERR_INVALID_ARG, "duplicate edge %d -> %d", src[ord[i]], dst[ord[i]]);
  std::fill(a_rowptr, a_rowptr + N + 1, 0);
  for (int64_t i = 0; i < nnz; ++i) {
    int64_t e = ord[i];
    a_rowptr[src[e] + 1]++;
    a_col[i] = dst[e];
    Pf_val[i] = float(double(w[e]) * inv(d_out[src[e]]));   // P_f[i][j]   = A[i][j] / d_out[i]
    PbT_val[i] = float(double(w[e]) * inv(d_in[dst[e]]));   // P_b^T[i][j] = A[i][j] / d_in[j]
  }
  for (int i = 0; i < N; ++i) a_rowptr[i + 1] += a_rowptr[i];

  // pattern(A^T): order edges by (dst, src)
  std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
    return dst[a] != dst[b] ? dst[a] < dst[b] : src[a] < src[b];
  });
  std::fill(at_rowptr, at_rowptr + N + 1, 0);
  for (int64_t i = 0; i < nnz; ++i) {
    int64_t e = ord[i];
    at_rowptr[dst[e] + 1]++;
    at_col[i] = src[e];
    Pb_val[i] = float(double(w[e]) * inv(d_in[dst[e]]));    // P_b[i][j]   = A[j][i] / d_in[i]
    PfT_val[i] = float(double(w[e]) * inv(d_out[src[e]]));  // P_f^T[i][j] = A[j][i] / d_out[j]
  }
  for (int i = 0; i < N; ++i) at_rowptr[i + 1] += at_rowptr[i];
  return PGTI_OK;
}

// Shared-memory staging plan of the diffusion SpMM (K2) on one CSR pattern: rows are cut into
// windows of `rows_per_window` consecutive nodes; window w stages the union of its rows' column
// indices (ascending, win_nodes[win_ptr[w] .. win_ptr[w+1])) and every CSR entry gets its column's
// position in that union (lcol).  Pure index bookkeeping: values and summation order unchanged.
extern "C" pgti_status pgti_graph_windows(int32_t N, const int32_t *rowptr, const int32_t *col,
                                          int32_t rows_per_window, int32_t *win_ptr,
                                          int32_t *win_nodes, uint16_t *lcol,
                                          int32_t *max_union) {
  pgti::clear_error();
  PGTI_REQUIRE(N > 0 && rowptr && win_ptr && max_union, PGTI_ERR_INVALID_ARG,
               "pgti_graph_windows: null pointer or N=%d", N);
  PGTI_REQUIRE(rows_per_window >= 1 && rows_per_window <= 64, PGTI_ERR_INVALID_ARG,
               "pgti_graph_windows: rows_per_window=%d outside [1, 64]", rows_per_window);
  const int64_t nnz = rowptr[N];
  PGTI_REQUIRE(rowptr[0] == 0 && nnz >= 0 && (nnz == 0 || (col && win_nodes && lcol)),
               PGTI_ERR_INVALID_ARG, "pgti_graph_windows: bad rowptr / null arrays");
  for (int32_t i = 0; i < N; ++i)
    PGTI_REQUIRE(rowptr[i + 1] >= rowptr[i], PGTI_ERR_INVALID_ARG, "rowptr not monotone at %d", i);
  const int32_t nwin = (N + rows_per_window - 1) / rows_per_window;
  std::vector<int32_t> u;
  int64_t pos = 0;
  int32_t mx = 0;
  win_ptr[0] = 0;
  for (int32_t w = 0; w < nwin; ++w) {
    const int32_t r0 = w * rows_per_window, r1 = std::min(N, r0 + rows_per_window);
    u.assign(col + rowptr[r0], col + rowptr[r1]);
    for (int32_t c : u)
      PGTI_REQUIRE(c >= 0 && c < N, PGTI_ERR_INVALID_ARG, "column %d outside [0, %d)", c, N);
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    PGTI_REQUIRE(u.size() <= 65535, PGTI_ERR_INVALID_ARG, "window %d union %zu > 65535", w,
                 u.size());
    for (int64_t e = rowptr[r0]; e < rowptr[r1]; ++e)
      lcol[e] = uint16_t(std::lower_bound(u.begin(), u.end(), col[e]) - u.begin());
    std::copy(u.begin(), u.end(), win_nodes + pos);
    pos += int64_t(u.size());
    win_ptr[w + 1] = int32_t(pos);
    mx = std::max(mx, int32_t(u.size()));
  }
  *max_union = mx;
  return PGTI_OK;
}

