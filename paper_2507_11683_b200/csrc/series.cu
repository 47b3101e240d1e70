// The HBM-resident series and index batching:
//   pgti_load_series     -- one consolidated H2D copy into a 16-byte-pitched buffer
//   pgti_series_stats    -- window-weighted Alg. 1 statistics, float64
//   pgti_series_normalize-- K0: in-place IEEE fp32 z-score
//   pgti_make_index      -- K_idx: Philox4x32-10 keys + stable radix sort
//   pgti_gather_batch    -- K1: window gather, one contiguous slab per sample
#include <cub/device/device_radix_sort.cuh>

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "profile.cuh"

struct pgti_series {
  int64_t row0, nrows, N, F, ld;
  float *buf;
};

namespace {

// ------------------------------------------------------------------ K0 pads / normalize
// One float4 per thread-iteration; rows are 16-byte aligned because ld % 4 == 0.
__global__ void k_zero_pads(float *__restrict__ buf, int64_t nrows, int64_t ld, int64_t nf) {
  const int64_t pad = ld - nf;
  const int64_t total = nrows * pad;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    int64_t r = i / pad, c = nf + i % pad;
    buf[r * ld + c] = 0.0f;
  }
}

__global__ void k_normalize(float *__restrict__ buf, int64_t nrows, int64_t ld, int64_t nf,
                            float mu, float sigma) {
  const int64_t q = ld / 4;
  const int64_t total = nrows * q;
  float4 *b4 = reinterpret_cast<float4 *>(buf);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c0 = (i % q) * 4;
    float4 v = b4[i];
    // IEEE round-to-nearest sub then div, no contraction: fl32(fl32(v - mu) / sigma)
    v.x = (c0 + 0 < nf) ? __fdiv_rn(__fsub_rn(v.x, mu), sigma) : 0.0f;
    v.y = (c0 + 1 < nf) ? __fdiv_rn(__fsub_rn(v.y, mu), sigma) : 0.0f;
    v.z = (c0 + 2 < nf) ? __fdiv_rn(__fsub_rn(v.z, mu), sigma) : 0.0f;
    v.w = (c0 + 3 < nf) ? __fdiv_rn(__fsub_rn(v.w, mu), sigma) : 0.0f;
    b4[i] = v;
  }
}

// ------------------------------------------------------------------ stats (float64)
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Each block takes rows; w(t) = #training windows whose x slice covers global row t.
__global__ void k_stats(const float *__restrict__ buf, int64_t row0, int64_t ld, int64_t nf,
                        int64_t row_lo, int64_t row_hi, int64_t S_tr, int T_in, double shift,
                        double *__restrict__ sums) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int64_t t = row_lo + blockIdx.x; t < row_hi; t += gridDim.x) {
    int64_t hi = t < S_tr - 1 ? t : S_tr - 1;
    int64_t lo = t - T_in + 1 > 0 ? t - T_in + 1 : 0;
    int64_t w = hi - lo + 1;
    if (w <= 0) continue;
    const float *row = buf + (t - row0) * ld;
    double a1 = 0.0, a2 = 0.0;
    for (int64_t c = threadIdx.x; c < nf; c += blockDim.x) {
      double d = double(row[c]) - shift;
      a1 += d;
      a2 += d * d;
    }
    s1 += double(w) * a1;
    s2 += double(w) * a2;
    if (threadIdx.x == 0) s0 += double(w) * double(nf);
  }
  __shared__ double red[3][32];
  s0 = warp_sum(s0);
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[0][wid] = s0, red[1][wid] = s1, red[2][wid] = s2;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    s0 = lane < nw ? red[0][lane] : 0.0;
    s1 = lane < nw ? red[1][lane] : 0.0;
    s2 = lane < nw ? red[2][lane] : 0.0;
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      atomicAdd(&sums[0], s0);
      atomicAdd(&sums[1], s1);
      atomicAdd(&sums[2], s2);
    }
  }
}

// ------------------------------------------------------------------ K_idx (Philox4x32-10)
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) k0 += W0, k1 += W1;
    const uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
    const uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0, c[1] = lo1, c[2] = n2, c[3] = lo0;
  }
}

__global__ void k_keys(int64_t n, int32_t win_lo, uint64_t seed, uint64_t epoch, uint32_t rank,
                       int shuffle, unsigned long long *__restrict__ keys,
                       int32_t *__restrict__ vals) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint32_t c[4] = {uint32_t(i), uint32_t(epoch), uint32_t(epoch >> 32), rank};
    philox4x32_10(c, uint32_t(seed), uint32_t(seed >> 32));
    if (keys) keys[i] = (static_cast<unsigned long long>(c[0]) << 32) | c[1];
    vals[i] = win_lo + int32_t(i);
    (void)shuffle;
  }
}

// batch-level shuffle (shuffle = 2): window t of the plan = win_lo + order[t / B] * B + t % B
__global__ void k_expand_batches(int64_t n_used, int B, int32_t win_lo,
                                 const int32_t *__restrict__ order, int32_t *__restrict__ idx) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n_used;
       t += int64_t(gridDim.x) * blockDim.x)
    idx[t] = win_lo + order[t / B] * B + int32_t(t % B);
}

// ------------------------------------------------------------------ K1 window gather
// LDG.128/STG.128 variant: block (chunk, b); each thread moves kUnroll float4 with all loads
// issued before the stores (bytes in flight).
constexpr int kGatherThreads = 256, kGatherUnroll = 4;

__global__ void __launch_bounds__(kGatherThreads)
    k_gather_ldg(const float4 *__restrict__ series, int64_t row0, int64_t nrows, int64_t ld4,
                 const int32_t *__restrict__ idx, int T_in, int T_out, float4 *__restrict__ x,
                 float4 *__restrict__ y, unsigned *__restrict__ err) {
  const int b = blockIdx.y;
  const int64_t s = int64_t(idx[b]) - row0;
  if (s < 0 || s + T_in + T_out > nrows) {
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicOr(err, pgti::kDevErrRange);
    return;
  }
  const int64_t nx = int64_t(T_in) * ld4, ny = int64_t(T_out) * ld4, tot = nx + ny;
  const float4 *src = series + s * ld4;
  float4 *xb = x + int64_t(b) * nx;
  float4 *yb = y + int64_t(b) * ny;
  const int64_t per_block = int64_t(kGatherThreads) * kGatherUnroll;
  for (int64_t base = int64_t(blockIdx.x) * per_block; base < tot;
       base += int64_t(gridDim.x) * per_block) {
    float4 v[kGatherUnroll];
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) {
      int64_t e = base + u * kGatherThreads + threadIdx.x;
      if (e < tot) v[u] = __ldg(src + e);
    }
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) {
      int64_t e = base + u * kGatherThreads + threadIdx.x;
      if (e < tot) {
        if (e < nx)
          __stcs(xb + e, v[u]);
        else
          __stcs(yb + (e - nx), v[u]);
      }
    }
  }
}

// TMA (bulk-copy engine) variant: each CTA moves one <= kChunk-byte piece of a sample's
// slab global -> smem (cp.async.bulk, mbarrier complete_tx) -> global (bulk store).
// The x/y split point (T_in*ld floats) is a multiple of 16 bytes, so pieces never straddle it
// when chunks are aligned to it: pieces are cut separately from the x and y parts.
constexpr int kChunk = 32768;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(32)
    k_gather_tma(const float *__restrict__ series, int64_t row0, int64_t nrows, int64_t ld,
                 const int32_t *__restrict__ idx, int T_in, int T_out, float *__restrict__ x,
                 float *__restrict__ y, int64_t xchunks, int64_t ychunks,
                 unsigned *__restrict__ err) {
  __shared__ alignas(128) unsigned char buf[kChunk];
  __shared__ alignas(8) uint64_t bar;
  const int b = blockIdx.y;
  const int64_t s = int64_t(idx[b]) - row0;
  if (s < 0 || s + T_in + T_out > nrows) {
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicOr(err, pgti::kDevErrRange);
    return;
  }
  if (threadIdx.x != 0) return;
  const int64_t xbytes = int64_t(T_in) * ld * 4, ybytes = int64_t(T_out) * ld * 4;
  const int64_t c = blockIdx.x;
  const char *src;
  char *dst;
  int64_t off, total;
  if (c < xchunks) {
    off = c * kChunk, total = xbytes;
    src = reinterpret_cast<const char *>(series + s * ld) + off;
    dst = reinterpret_cast<char *>(x) + int64_t(b) * xbytes + off;
  } else {
    off = (c - xchunks) * kChunk, total = ybytes;
    if (c - xchunks >= ychunks) return;
    src = reinterpret_cast<const char *>(series + (s + T_in) * ld) + off;
    dst = reinterpret_cast<char *>(y) + int64_t(b) * ybytes + off;
  }
  const uint32_t bytes = uint32_t(total - off < kChunk ? total - off : kChunk);
  const uint32_t sb = smem_u32(buf), mb = smem_u32(&bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(sb),
      "l"(src), "r"(bytes), "r"(mb)
      : "memory");
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(mb)
        : "memory");
  }
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(sb),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// K1 variant: PGTI_GATHER=tma selects the bulk-copy (TMA engine) kernel, default LDG/STG.128.
// Read per call (host-side, cheap) so a process can compare both.
int gather_mode() {
  const char *e = getenv("PGTI_GATHER");
  return (e && strcmp(e, "tma") == 0) ? 1 : 0;
}

}  // namespace

// =========================================================================== C ABI
extern "C" pgti_status pgti_load_series(pgti_series **out, const float *host_rows, int64_t row0,
                                        int64_t nrows, int64_t N, int64_t F, float *dev_buf,
                                        int64_t ld, void *stream) {
  pgti::clear_error();
  PGTI_REQUIRE(out && host_rows && dev_buf, PGTI_ERR_INVALID_ARG, "pgti_load_series: null pointer");
  PGTI_REQUIRE(row0 >= 0 && nrows > 0 && N > 0 && F > 0, PGTI_ERR_INVALID_ARG,
               "pgti_load_series: row0=%lld nrows=%lld N=%lld F=%lld", (long long)row0,
               (long long)nrows, (long long)N, (long long)F);
  PGTI_REQUIRE(ld >= N * F && ld % 4 == 0, PGTI_ERR_ALIGNMENT,
               "pgti_load_series: ld=%lld must be >= N*F=%lld and a multiple of 4", (long long)ld,
               (long long)(N * F));
  PGTI_REQUIRE(pgti::aligned16(dev_buf), PGTI_ERR_ALIGNMENT, "dev_buf not 16-byte aligned");
  cudaStream_t s = pgti::as_stream(stream);
  const size_t row_bytes = size_t(N * F) * 4;
  PGTI_CUDA_TRY(cudaMemcpy2DAsync(dev_buf, size_t(ld) * 4, host_rows, row_bytes, row_bytes,
                                  size_t(nrows), cudaMemcpyHostToDevice, s));
  if (ld > N * F) {
    int64_t total = nrows * (ld - N * F);
    int grid = int(std::min<int64_t>(pgti::ceil_div(total, 256), 4 * 148 * 8));
    pgti::ProfScope prof(pgti::kProfSeries, s, 4.0 * double(total), 0.0);
    k_zero_pads<<<grid, 256, 0, s>>>(dev_buf, nrows, ld, N * F);
    PGTI_LAUNCH_TRY();
  }
  auto *h = new pgti_series{row0, nrows, N, F, ld, dev_buf};
  *out = h;
  return PGTI_OK;
}

extern "C" pgti_status pgti_series_stats(const pgti_series *sr, int64_t S_tr, int T_in,
                                         int64_t row_lo, int64_t row_hi, double shift,
                                         double *dev_sums, void *stream) {
  pgti::clear_error();
  PGTI_REQUIRE(sr && dev_sums, PGTI_ERR_INVALID_ARG, "pgti_series_stats: null pointer");
  PGTI_REQUIRE(S_tr >= 1 && T_in >= 1 && std::isfinite(shift), PGTI_ERR_INVALID_ARG,
               "pgti_series_stats: S_tr=%lld T_in=%d", (long long)S_tr, T_in);
  PGTI_REQUIRE(row_lo >= sr->row0 && row_hi <= sr->row0 + sr->nrows && row_lo <= row_hi,
               PGTI_ERR_OUT_OF_RANGE, "pgti_series_stats: rows [%lld,%lld) not inside held [%lld,%lld)",
               (long long)row_lo, (long long)row_hi, (long long)sr->row0,
               (long long)(sr->row0 + sr->nrows));
  if (row_hi == row_lo) return PGTI_OK;
  int grid = int(std::min<int64_t>(row_hi - row_lo, 148 * 16));
  pgti::ProfScope prof(pgti::kProfSeries, pgti::as_stream(stream),
                       4.0 * double(row_hi - row_lo) * double(sr->N * sr->F), 0.0);
  k_stats<<<grid, 256, 0, pgti::as_stream(stream)>>>(sr->buf, sr->row0, sr->ld, sr->N * sr->F,
                                                      row_lo, row_hi, S_tr, T_in, shift, dev_sums);
  PGTI_LAUNCH_TRY();
  return PGTI_OK;
}

extern "C" pgti_status pgti_series_normalize(pgti_series *sr, double mu, double sigma,
                                             void *stream) {
  pgti::clear_error();
  PGTI_REQUIRE(sr, PGTI_ERR_INVALID_ARG, "pgti_series_normalize: null series");
  PGTI_REQUIRE(std::isfinite(mu), PGTI_ERR_NONFINITE, "mu=%g not finite", mu);
  PGTI_REQUIRE(std::isfinite(sigma) && sigma > 0.0 && float(sigma) > 0.f, PGTI_ERR_ZERO_VARIANCE,
               "sigma=%g must be finite and > 0", sigma);
  int64_t total = sr->nrows * (sr->ld / 4);
  int grid = int(std::min<int64_t>(pgti::ceil_div(total, 256), 148 * 16));
  pgti::ProfScope prof(pgti::kProfSeries, pgti::as_stream(stream), 8.0 * double(total) * 4, 0.0);
  k_normalize<<<grid, 256, 0, pgti::as_stream(stream)>>>(sr->buf, sr->nrows, sr->ld,
                                                          sr->N * sr->F, float(mu), float(sigma));
  PGTI_LAUNCH_TRY();
  return PGTI_OK;
}

namespace pgti {
void series_view(const pgti_series *sr, const float **buf, int64_t *row0, int64_t *nrows,
                 int64_t *N, int64_t *F, int64_t *ld) {
  *buf = sr->buf, *row0 = sr->row0, *nrows = sr->nrows, *N = sr->N, *F = sr->F, *ld = sr->ld;
}
}  // namespace pgti

extern "C" pgti_status pgti_series_info(const pgti_series *sr, int64_t *row0, int64_t *nrows,
                                        int64_t *N, int64_t *F, int64_t *ld) {
  pgti::clear_error();
  PGTI_REQUIRE(sr, PGTI_ERR_INVALID_ARG, "pgti_series_info: null series");
  if (row0) *row0 = sr->row0;
  if (nrows) *nrows = sr->nrows;
  if (N) *N = sr->N;
  if (F) *F = sr->F;
  if (ld) *ld = sr->ld;
  return PGTI_OK;
}

extern "C" pgti_status pgti_series_destroy(pgti_series *sr) {
  pgti::clear_error();
  delete sr;
  return PGTI_OK;
}

extern "C" pgti_status pgti_make_index(const pgti_series *sr, int64_t win_lo, int64_t win_hi,
                                       int T_in, int T_out, int B, uint64_t seed, uint64_t epoch,
                                       int rank, int shuffle, int32_t *dev_idx, int64_t *n_used,
                                       void *stream) {
  pgti::clear_error();
  PGTI_REQUIRE(sr && dev_idx && n_used, PGTI_ERR_INVALID_ARG, "pgti_make_index: null pointer");
  PGTI_REQUIRE(T_in >= 1 && T_out >= 1 && B >= 1 && rank >= 0 && shuffle >= 0 && shuffle <= 2,
               PGTI_ERR_INVALID_ARG, "pgti_make_index: T_in=%d T_out=%d B=%d rank=%d shuffle=%d",
               T_in, T_out, B, rank, shuffle);
  PGTI_REQUIRE(win_lo >= 0 && win_hi >= win_lo && win_hi < (int64_t(1) << 31),
               PGTI_ERR_INVALID_ARG, "pgti_make_index: windows [%lld,%lld)", (long long)win_lo,
               (long long)win_hi);
  PGTI_REQUIRE(sr->nrows >= T_in + T_out, PGTI_ERR_TOO_FEW_ENTRIES,
               "series holds %lld rows < T_in+T_out=%d", (long long)sr->nrows, T_in + T_out);
  PGTI_REQUIRE(win_lo >= sr->row0 && (win_hi == win_lo ||
                                      win_hi - 1 + T_in + T_out <= sr->row0 + sr->nrows),
               PGTI_ERR_OUT_OF_RANGE,
               "windows [%lld,%lld) need rows up to %lld; series holds [%lld,%lld)",
               (long long)win_lo, (long long)win_hi, (long long)(win_hi - 1 + T_in + T_out),
               (long long)sr->row0, (long long)(sr->row0 + sr->nrows));
  const int64_t n = win_hi - win_lo;
  PGTI_REQUIRE(n >= B, PGTI_ERR_TOO_FEW_WINDOWS, "%lld windows < batch %d", (long long)n, B);
  cudaStream_t s = pgti::as_stream(stream);
  const int grid = int(std::min<int64_t>(pgti::ceil_div(n, 256), 148 * 8));
  pgti::ProfScope prof(pgti::kProfIndex, s, double(n) * (shuffle ? 48.0 : 4.0), 0.0,
                       shuffle ? 5 : 1);
  if (shuffle == 2) {  // membership frozen, batch order permuted
    const int64_t nb = n / B;
    size_t temp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, (unsigned long long *)nullptr,
                                    (unsigned long long *)nullptr, (int32_t *)nullptr,
                                    (int32_t *)nullptr, int(nb), 0, 64, s);
    const size_t kb = pgti::round_up(nb * 8, 256), vb = pgti::round_up(nb * 4, 256);
    char *scratch = nullptr;
    PGTI_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&scratch), 2 * kb + 2 * vb + temp_bytes,
                                  s));
    auto *keys_in = reinterpret_cast<unsigned long long *>(scratch);
    auto *keys_out = reinterpret_cast<unsigned long long *>(scratch + kb);
    auto *vals_in = reinterpret_cast<int32_t *>(scratch + 2 * kb);
    auto *vals_out = reinterpret_cast<int32_t *>(scratch + 2 * kb + vb);
    void *temp = scratch + 2 * kb + 2 * vb;
    const int gb = int(std::min<int64_t>(pgti::ceil_div(nb, 256), 148 * 8));
    k_keys<<<gb, 256, 0, s>>>(nb, 0, seed, epoch, uint32_t(rank), 1, keys_in, vals_in);
    cudaError_t e1 = cudaGetLastError();
    cudaError_t e2 = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in,
                                                     vals_out, int(nb), 0, 64, s);
    k_expand_batches<<<grid, 256, 0, s>>>(nb * B, B, int32_t(win_lo), vals_out, dev_idx);
    cudaError_t e3 = cudaGetLastError();
    cudaError_t e4 = cudaFreeAsync(scratch, s);
    PGTI_CUDA_TRY(e1);
    PGTI_CUDA_TRY(e2);
    PGTI_CUDA_TRY(e3);
    PGTI_CUDA_TRY(e4);
  } else if (!shuffle) {
    k_keys<<<grid, 256, 0, s>>>(n, int32_t(win_lo), seed, epoch, uint32_t(rank), 0, nullptr,
                                dev_idx);
    PGTI_LAUNCH_TRY();
  } else {
    size_t temp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, (unsigned long long *)nullptr,
                                    (unsigned long long *)nullptr, (int32_t *)nullptr,
                                    (int32_t *)nullptr, int(n), 0, 64, s);
    const size_t kb = pgti::round_up(n * 8, 256), vb = pgti::round_up(n * 4, 256);
    char *scratch = nullptr;
    PGTI_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&scratch), 2 * kb + vb + temp_bytes, s));
    auto *keys_in = reinterpret_cast<unsigned long long *>(scratch);
    auto *keys_out = reinterpret_cast<unsigned long long *>(scratch + kb);
    auto *vals_in = reinterpret_cast<int32_t *>(scratch + 2 * kb);
    void *temp = scratch + 2 * kb + vb;
    k_keys<<<grid, 256, 0, s>>>(n, int32_t(win_lo), seed, epoch, uint32_t(rank), 1, keys_in,
                                vals_in);
    cudaError_t e1 = cudaGetLastError();
    cudaError_t e2 = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in,
                                                     dev_idx, int(n), 0, 64, s);
    cudaError_t e3 = cudaFreeAsync(scratch, s);
    PGTI_CUDA_TRY(e1);
    PGTI_CUDA_TRY(e2);
    PGTI_CUDA_TRY(e3);
  }
  *n_used = (n / B) * B;
  return PGTI_OK;
}

extern "C" pgti_status pgti_gather_batch(const pgti_series *sr, const int32_t *dev_idx, int B,
                                         int T_in, int T_out, float *x, float *y, void *stream) {
  pgti::clear_error();
  PGTI_REQUIRE(sr && dev_idx && x && y, PGTI_ERR_INVALID_ARG, "pgti_gather_batch: null pointer");
  PGTI_REQUIRE(B >= 1 && T_in >= 1 && T_out >= 1, PGTI_ERR_INVALID_ARG,
               "pgti_gather_batch: B=%d T_in=%d T_out=%d", B, T_in, T_out);
  PGTI_REQUIRE(pgti::aligned16(x) && pgti::aligned16(y), PGTI_ERR_ALIGNMENT,
               "x / y must be 16-byte aligned");
  unsigned *err = pgti::device_error_flag();
  PGTI_REQUIRE(err, PGTI_ERR_CUDA, "device error flag unavailable");
  cudaStream_t s = pgti::as_stream(stream);
  // algorithmic bytes: 2 B (T_in+T_out) N F 4 -- read + write, pads excluded
  pgti::ProfScope prof(pgti::kProfGather, s, 8.0 * B * (T_in + T_out) * double(sr->N * sr->F),
                       0.0);
  if (gather_mode() == 1) {
    const int64_t xb = int64_t(T_in) * sr->ld * 4, yb = int64_t(T_out) * sr->ld * 4;
    const int64_t xc = pgti::ceil_div(xb, kChunk), yc = pgti::ceil_div(yb, kChunk);
    dim3 grid(unsigned(xc + yc), unsigned(B));
    k_gather_tma<<<grid, 32, 0, s>>>(sr->buf, sr->row0, sr->nrows, sr->ld, dev_idx, T_in, T_out,
                                     x, y, xc, yc, err);
  } else {
    const int64_t tot4 = int64_t(T_in + T_out) * (sr->ld / 4);
    const int64_t per_block = int64_t(kGatherThreads) * kGatherUnroll;
    dim3 grid(unsigned(pgti::ceil_div(tot4, per_block)), unsigned(B));
    k_gather_ldg<<<grid, kGatherThreads, 0, s>>>(
        reinterpret_cast<const float4 *>(sr->buf), sr->row0, sr->nrows, sr->ld / 4, dev_idx, T_in,
        T_out, reinterpret_cast<float4 *>(x), reinterpret_cast<float4 *>(y), err);
  }
  PGTI_LAUNCH_TRY();
  return PGTI_OK;
}
