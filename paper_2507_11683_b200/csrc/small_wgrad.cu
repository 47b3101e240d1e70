// Skinny weight gradients (bias rows, layer-0 input rows, readout W_out / b_out):
// out[s][j] = sum_t sum_r S_t[r][s] G_t[r][j] with ns <= 12 small rows and a wide G.
// Memory-bound on G (read once, coalesced along j); the small operand is staged per 64-row tile
// in shared memory and broadcast.  Row chunks never cross a time step; chunk partials are summed
// in a fixed order (bitwise reproducible).
#include "kernels.cuh"
#include "profile.cuh"

namespace pgti {
namespace {

constexpr int kSmallMax = 12, kTile = 64, kThr = 256;

struct Plan {
  int ns, ngt, RC, cpt, nchunks;
};

Plan plan_for(const SmallWgrad &p) {
  Plan q{};
  q.ns = p.mode == kSmallBiasX ? (p.Dx ? p.M * p.F : 0) + 1 : p.F_out;
  q.ngt = p.NG + (p.mode == kSmallReadout ? 1 : 0);
  const int64_t tr = int64_t(p.T) * p.R;
  q.RC = int(std::max<int64_t>(kTile, round_up(ceil_div(tr, 2 * kNumSMs * 2), kTile)));
  q.cpt = int(ceil_div(p.R, q.RC));
  q.nchunks = p.T * q.cpt;
  return q;
}

__global__ void __launch_bounds__(kThr) k_small_wgrad(const __grid_constant__ SmallWgrad p,
                                                      Plan q) {
  __shared__ float S[kTile][kSmallMax];
  __shared__ float red[kThr / 128][kSmallMax][129];
  griddep_launch_dependents();
  griddep_wait();
  const int chunk = blockIdx.x, t = chunk / q.cpt;
  const int r0 = (chunk - t * q.cpt) * q.RC, r1 = min(p.R, r0 + q.RC);
  const int j = threadIdx.x % 128, lg = threadIdx.x / 128;
  float acc[kSmallMax];
#pragma unroll
  for (int s = 0; s < kSmallMax; ++s) acc[s] = 0.f;
  const float *G = p.G + t * p.g_tstride;
  for (int rb = r0; rb < r1; rb += kTile) {
    const int nr = min(kTile, r1 - rb);
    for (int i = threadIdx.x; i < nr * q.ns; i += kThr) {
      const int rr = i / q.ns, s = i % q.ns, row = rb + rr;
      float v;
      if (p.mode == kSmallBiasX) {
        if (s == q.ns - 1) {
          v = 1.0f;
        } else {
          const int m = s / p.F, f = s % p.F;
          v = __ldg(p.Dx + m * p.dx_mstride + t * p.dx_tstride + int64_t(row) * p.F + f);
        }
      } else {
        v = __ldg(p.dy + (int64_t(t) * p.R + row) * p.F_out + s);
      }
      S[rr][s] = v;
    }
    __syncthreads();
    if (j < q.ngt)
      for (int rr = lg; rr < nr; rr += kThr / 128) {
        const float g = j < p.NG ? __ldg(G + int64_t(rb + rr) * p.NG + j) : 1.0f;
#pragma unroll
        for (int s = 0; s < kSmallMax; ++s)
          if (s < q.ns) acc[s] = fmaf(S[rr][s], g, acc[s]);
      }
    __syncthreads();
  }
#pragma unroll
  for (int s = 0; s < kSmallMax; ++s) red[lg][s][j] = acc[s];
  __syncthreads();
  if (lg == 0 && j < q.ngt)
    for (int s = 0; s < q.ns; ++s)
      p.partial[(int64_t(chunk) * q.ns + s) * q.ngt + j] = red[0][s][j] + red[1][s][j];
}

// bf16 G (the tensor-core path's gate gradients): thread = 2 adjacent columns (one 4-byte load),
// NG/2 threads per row, kThr/(NG/2) row groups, folded in shared memory in group order (fixed,
// deterministic).  No ones column (bias rows use S = 1 instead).
__global__ void __launch_bounds__(kThr) k_small_wgrad_bf(const __grid_constant__ SmallWgrad p,
                                                         Plan q) {
  __shared__ float S[kTile][kSmallMax];
  __shared__ float2 red[kSmallMax][64];
  griddep_launch_dependents();
  griddep_wait();
  const int chunk = blockIdx.x, t = chunk / q.cpt;
  const int r0 = (chunk - t * q.cpt) * q.RC, r1 = min(p.R, r0 + q.RC);
  const int cpr = p.NG / 2, ng = kThr / cpr;
  const int jj = threadIdx.x % cpr, lg = threadIdx.x / cpr;
  float2 acc[kSmallMax];
#pragma unroll
  for (int s = 0; s < kSmallMax; ++s) acc[s] = make_float2(0.f, 0.f);
  const __nv_bfloat162 *G =
      reinterpret_cast<const __nv_bfloat162 *>(p.Gb + t * p.g_tstride) + jj;
  for (int rb = r0; rb < r1; rb += kTile) {
    const int nr = min(kTile, r1 - rb);
    for (int i = threadIdx.x; i < nr * q.ns; i += kThr) {
      const int rr = i / q.ns, s = i % q.ns, row = rb + rr;
      float v;
      if (s == q.ns - 1) {
        v = 1.0f;
      } else {
        const int m = s / p.F, f = s % p.F;
        v = __ldg(p.Dx + m * p.dx_mstride + t * p.dx_tstride + int64_t(row) * p.F + f);
      }
      S[rr][s] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = lg; rr < nr; rr += ng) {
      const float2 g = __bfloat1622float2(G[int64_t(rb + rr) * cpr]);
#pragma unroll
      for (int s = 0; s < kSmallMax; ++s)
        if (s < q.ns) {
          const float v = S[rr][s];
          acc[s].x = fmaf(v, g.x, acc[s].x), acc[s].y = fmaf(v, g.y, acc[s].y);
        }
    }
    __syncthreads();
  }
  for (int g = 0; g < ng; ++g) {  // fold the row groups in order
    if (lg == g)
#pragma unroll
      for (int s = 0; s < kSmallMax; ++s) {
        if (g == 0) {
          red[s][jj] = acc[s];
        } else {
          const float2 o = red[s][jj];
          red[s][jj] = make_float2(o.x + acc[s].x, o.y + acc[s].y);
        }
      }
    __syncthreads();
  }
  float *out = p.partial + int64_t(chunk) * q.ns * q.ngt;
  for (int i = threadIdx.x; i < q.ns * cpr; i += kThr) {
    const int s = i / cpr, c = i % cpr;
    *reinterpret_cast<float2 *>(out + s * q.ngt + 2 * c) = red[s][c];
  }
}

// One warp per output: lane l sums chunks l, l+32, ... (fixed order), then a fixed xor-tree.
__global__ void k_small_reduce(const __grid_constant__ SmallWgrad p, Plan q) {
  griddep_launch_dependents();
  griddep_wait();
  const int n = q.ns * q.ngt;
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += (gridDim.x * blockDim.x) >> 5) {
    float sum = 0.f;
    for (int c = lane; c < q.nchunks; c += 32) sum += p.partial[int64_t(c) * n + i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane) continue;
    const int s = i / q.ngt, j = i % q.ngt;
    if (p.mode == kSmallBiasX) {
      const int row = s == q.ns - 1 ? p.M * p.C_in : (s / p.F) * p.C_in + s % p.F;
      p.out[int64_t(row) * p.NG + j] = sum;
    } else {
      // W_out[j][o] (j < H) followed by b_out[o] (the ones column j == H)
      p.out[int64_t(j) * p.F_out + s] = sum;
    }
  }
}

}  // namespace

size_t small_wgrad_partial_floats(int T, int R, int NG) {
  const int64_t tr = int64_t(T) * R;
  const int RC = int(std::max<int64_t>(kTile, round_up(ceil_div(tr, 2 * kNumSMs * 2), kTile)));
  return size_t(T) * size_t(ceil_div(R, RC)) * kSmallMax * size_t(NG + 1);
}

cudaError_t launch_small_wgrad(const SmallWgrad &p, cudaStream_t s) {
  const Plan q = plan_for(p);
  if (q.ns > kSmallMax || q.ngt > 128 || p.NG > 128) return cudaErrorInvalidValue;
  if (p.Gb && (p.mode != kSmallBiasX || p.NG % 64)) return cudaErrorInvalidValue;
  if (int64_t(q.nchunks) * q.ns * q.ngt > p.partial_cap) return cudaErrorInvalidValue;
  cudaError_t e;
  {
    const double tr = double(p.T) * p.R;
    ProfScope prof(kProfGemmWgrad, s, tr * ((p.Gb ? 2.0 : 4.0) * p.NG + 4.0 * q.ns),
                   2.0 * tr * q.ns * q.ngt);
    if (p.Gb)
      e = pdl_launch(k_small_wgrad_bf, dim3(unsigned(q.nchunks)), dim3(kThr), 0, s, p, q);
    else
      e = pdl_launch(k_small_wgrad, dim3(unsigned(q.nchunks)), dim3(kThr), 0, s, p, q);
  }
  if (e != cudaSuccess) return e;
  ProfScope prof(kProfReduce, s, 4.0 * double(q.nchunks + 1) * q.ns * q.ngt,
                 double(q.nchunks) * q.ns * q.ngt);
  return pdl_launch(k_small_reduce, dim3(unsigned(ceil_div(q.ns * q.ngt, 8))), dim3(256), 0, s,
                    p, q);
}

}  // namespace pgti
