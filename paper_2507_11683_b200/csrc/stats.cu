// Finalisation of Alg. 1's statistics and of the validation MAE, inside the library (the
// caller does no arithmetic on them):
//  * pgti_stats_finalize   -- the three window-weighted sums of pgti_series_stats -> mean,
//                             population variance (Alg. 1);
//  * pgti_series_moments   -- both passes of pgti_series_stats (shift 0, then shift = mean),
//                             the cross-rank NCCL sum of the partial sums (halo shards) and the
//                             finalisation: mu, sigma as Alg. 1 computes them over x_train;
//  * pgti_mean_losses      -- per-batch validation losses summed on the device in a fixed order,
//                             summed over ranks (the per-epoch validation AllReduce), and
//                             divided by the batch count.
#include <cmath>

#include "common.cuh"
#include "profile.cuh"

namespace {

// One CTA sums n floats in float64 in a fixed order (thread-strided partials, then a tree):
// bitwise reproducible for a given n.  acc[0] = sum, acc[1] = n.
__global__ void k_sum_f32(const float *__restrict__ v, int64_t n, double *__restrict__ acc) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += double(v[i]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) acc[0] = red[0], acc[1] = double(n);
}

}  // namespace

extern "C" pgti_status pgti_stats_finalize(const double sums[3], double shift, double *mean,
                                           double *var) {
  pgti::clear_error();
  PGTI_REQUIRE(sums && mean && var, PGTI_ERR_INVALID_ARG, "pgti_stats_finalize: null pointer");
  PGTI_REQUIRE(sums[0] > 0.0 && std::isfinite(sums[0]), PGTI_ERR_TOO_FEW_ENTRIES,
               "pgti_stats_finalize: weight sum s0=%g (no training window covers the rows)",
               sums[0]);
  PGTI_REQUIRE(std::isfinite(sums[1]) && std::isfinite(sums[2]) && std::isfinite(shift),
               PGTI_ERR_NONFINITE, "pgti_stats_finalize: s1=%g s2=%g shift=%g", sums[1], sums[2],
               shift);
  // Alg. 1: mean(x_train) = shift + E[v - shift]; line 202 (population std, ddof 0):
  // var = E[(v - shift)^2] - E[v - shift]^2, exact for any shift, cancellation-free when the
  // shift is the mean (second pass)
  const double d = sums[1] / sums[0];
  *mean = shift + d;
  const double v = sums[2] / sums[0] - d * d;
  *var = v > 0.0 ? v : 0.0;
  return PGTI_OK;
}

extern "C" pgti_status pgti_series_moments(const pgti_series *sr, int64_t S_tr, int T_in,
                                           int64_t row_lo, int64_t row_hi, pgti_comm *comm,
                                           double *dev_sums, double *mu, double *sigma,
                                           void *stream) {
  pgti::clear_error();
  PGTI_REQUIRE(sr && dev_sums && mu && sigma, PGTI_ERR_INVALID_ARG,
               "pgti_series_moments: null pointer");
  cudaStream_t s = pgti::as_stream(stream);
  double shift = 0.0, mean = 0.0, var = 0.0;
  for (int pass = 0; pass < 2; ++pass) {
    double h[3];
    PGTI_CUDA_TRY(cudaMemsetAsync(dev_sums, 0, 3 * sizeof(double), s));
    PGTI_STATUS_TRY(pgti_series_stats(sr, S_tr, T_in, row_lo, row_hi, shift, dev_sums, stream));
    if (comm) PGTI_STATUS_TRY(pgti_allreduce_f64(comm, dev_sums, 3, stream));
    PGTI_CUDA_TRY(cudaMemcpyAsync(h, dev_sums, sizeof h, cudaMemcpyDeviceToHost, s));
    PGTI_CUDA_TRY(cudaStreamSynchronize(s));
    PGTI_STATUS_TRY(pgti_stats_finalize(h, shift, &mean, &var));
    shift = mean;
  }
  *mu = mean;
  *sigma = std::sqrt(var);
  PGTI_REQUIRE(*sigma > 0.0, PGTI_ERR_ZERO_VARIANCE,
               "pgti_series_moments: sigma = 0 over the training windows (S:150)");
  return PGTI_OK;
}

extern "C" pgti_status pgti_mean_losses(pgti_comm *comm, const float *dev_losses, int64_t n,
                                        double *dev_scratch, double *mean, void *stream) {
  pgti::clear_error();
  PGTI_REQUIRE(dev_scratch && mean && (dev_losses || n == 0) && n >= 0, PGTI_ERR_INVALID_ARG,
               "pgti_mean_losses: null pointer or n=%lld", (long long)n);
  cudaStream_t s = pgti::as_stream(stream);
  if (n > 0) {
    pgti::ProfScope prof(pgti::kProfLoss, s, 4.0 * double(n), double(n));
    k_sum_f32<<<1, 256, 0, s>>>(dev_losses, n, dev_scratch);
    PGTI_LAUNCH_TRY();
  } else {
    PGTI_CUDA_TRY(cudaMemsetAsync(dev_scratch, 0, 2 * sizeof(double), s));
  }
  if (comm) PGTI_STATUS_TRY(pgti_allreduce_f64(comm, dev_scratch, 2, stream));
  double h[2];
  PGTI_CUDA_TRY(cudaMemcpyAsync(h, dev_scratch, sizeof h, cudaMemcpyDeviceToHost, s));
  PGTI_CUDA_TRY(cudaStreamSynchronize(s));
  *mean = h[1] > 0.0 ? h[0] / h[1] : std::nan("");
  return PGTI_OK;
}
