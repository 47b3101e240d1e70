// K2: CSR SpMM for the diffusion convolution (Li et al. Eq. 2 [ext]).
// Dense operand layout [G][N][W]: node-major, every node's W = B*C values contiguous, so one
// CSR row of the transition matrix multiplies whole 512-byte warp-wide slices.
// Warp-per-(row, 128-column chunk): the row's (col, val) pairs are fetched once per warp into
// registers and broadcast with shuffles; the neighbour slices are read with 128-bit loads,
// kUnroll of them in flight; fp32 accumulation in CSR order (deterministic).
#include "kernels.cuh"
#include "profile.cuh"

namespace pgti {
namespace {

struct SpmmParams {
  SpmmJob job[kMaxSpmmJobs];
  int njobs;
  int N;
  int64_t total_warps;
};

template <int VEC>
struct VecT;
template <>
struct VecT<4> {
  using T = float4;
};
template <>
struct VecT<1> {
  using T = float;
};

__device__ __forceinline__ void fma_v(float4 &a, float s, const float4 &x) {
  a.x = fmaf(s, x.x, a.x);
  a.y = fmaf(s, x.y, a.y);
  a.z = fmaf(s, x.z, a.z);
  a.w = fmaf(s, x.w, a.w);
}
__device__ __forceinline__ void fma_v(float &a, float s, const float &x) { a = fmaf(s, x, a); }
__device__ __forceinline__ void add_v(float4 &a, const float4 &x) {
  a.x += x.x, a.y += x.y, a.z += x.z, a.w += x.w;
}
__device__ __forceinline__ void add_v(float &a, const float &x) { a += x; }
__device__ __forceinline__ void zero_v(float4 &a) { a = make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void zero_v(float &a) { a = 0.f; }

template <int VEC>
__global__ void __launch_bounds__(256) k_spmm(const __grid_constant__ SpmmParams p) {
  using V = typename VecT<VEC>::T;
  const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= p.total_warps) return;
  int j = 0;
#pragma unroll
  for (int q = 1; q < kMaxSpmmJobs; ++q)
    if (q < p.njobs && wid >= p.job[q].warp_begin) j = q;
  const SpmmJob &jb = p.job[j];
  int64_t rem = wid - jb.warp_begin;
  const int64_t per_group = int64_t(p.N) * jb.chunks;
  const int64_t g = rem / per_group;
  rem -= g * per_group;
  const int n = int(rem / jb.chunks);
  const int64_t ch = rem - int64_t(n) * jb.chunks;
  const int64_t col0 = ch * (32 * VEC) + lane * VEC;
  const bool active = col0 < jb.W;
  const int64_t goff = g * jb.gstride;

  V acc;
  zero_v(acc);
  for (int t = 0; t < jb.nterms; ++t) {
    const int32_t beg = jb.rowptr[t][n], end = jb.rowptr[t][n + 1];
    const float *X = jb.X[t] + goff;
    for (int32_t e0 = beg; e0 < end; e0 += 32) {
      const int cnt = min(32, end - e0);
      int32_t mycol = 0;
      float myval = 0.f;
      if (lane < cnt) mycol = __ldg(jb.col[t] + e0 + lane), myval = __ldg(jb.val[t] + e0 + lane);
      int e = 0;
      for (; e + 4 <= cnt; e += 4) {
        V xv[4];
        float vv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = __shfl_sync(0xffffffffu, mycol, e + u);
          vv[u] = __shfl_sync(0xffffffffu, myval, e + u);
          if (active) xv[u] = __ldg(reinterpret_cast<const V *>(X + int64_t(c) * jb.W + col0));
        }
        if (active) {
#pragma unroll
          for (int u = 0; u < 4; ++u) fma_v(acc, vv[u], xv[u]);
        }
      }
      for (; e < cnt; ++e) {
        const int c = __shfl_sync(0xffffffffu, mycol, e);
        const float v = __shfl_sync(0xffffffffu, myval, e);
        if (active) fma_v(acc, v, __ldg(reinterpret_cast<const V *>(X + int64_t(c) * jb.W + col0)));
      }
    }
  }
  if (!active) return;
  const int64_t o = goff + int64_t(n) * jb.W + col0;
  if (jb.add) add_v(acc, *reinterpret_cast<const V *>(jb.add + o));
  V *Y = reinterpret_cast<V *>(jb.Y + o);
  if (jb.accumulate) add_v(acc, *Y);
  *Y = acc;
}

}  // namespace

cudaError_t launch_spmm(SpmmJob *jobs, int njobs, int N, cudaStream_t s) {
  if (njobs <= 0) return cudaSuccess;
  if (njobs > kMaxSpmmJobs) return cudaErrorInvalidValue;
  bool vec4 = true;
  for (int i = 0; i < njobs; ++i) {
    const SpmmJob &j = jobs[i];
    auto al = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    vec4 = vec4 && j.W % 4 == 0 && j.gstride % 4 == 0 && al(j.Y) && (!j.add || al(j.add)) &&
           al(j.X[0]) && (j.nterms < 2 || al(j.X[1]));
  }
  const int vw = vec4 ? 128 : 32;
  SpmmParams p{};
  int64_t w = 0;
  for (int i = 0; i < njobs; ++i) {
    p.job[i] = jobs[i];
    p.job[i].chunks = ceil_div(jobs[i].W, vw);
    p.job[i].warp_begin = w;
    w += int64_t(jobs[i].G) * N * p.job[i].chunks;
  }
  p.njobs = njobs;
  p.N = N;
  p.total_warps = w;
  if (w == 0) return cudaSuccess;
  // algorithmic bytes (SURVEY 8(d) K2 model): each dense operand row read once per term,
  // output written once, addend / accumulator read once, CSR (col, val, rowptr) once per group
  double bytes = 0.0, flops = 0.0;
  for (int i = 0; i < njobs; ++i) {
    const SpmmJob &j = jobs[i];
    const double nw = double(N) * double(j.W) * 4.0 * j.G;
    bytes += nw * (1 + j.nterms + (j.add ? 1 : 0) + (j.accumulate ? 1 : 0));
    for (int t = 0; t < j.nterms; ++t) {
      bytes += (double(j.nnz[t]) * 8.0 + double(N + 1) * 4.0) * j.G;
      flops += 2.0 * double(j.nnz[t]) * double(j.W) * j.G;
    }
  }
  ProfScope prof(kProfSpmm, s, bytes, flops);
  const int64_t blocks = ceil_div(w, 8);
  if (vec4)
    k_spmm<4><<<unsigned(blocks), 256, 0, s>>>(p);
  else
    k_spmm<1><<<unsigned(blocks), 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace pgti
