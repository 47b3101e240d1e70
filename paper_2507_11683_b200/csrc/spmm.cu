// K2: CSR SpMM for the diffusion convolution (Li et al. Eq. 2 [ext]).
// Dense operand layout [G][N][W]: node-major, every node's W = B*C values contiguous, so one
// CSR row of the transition matrix multiplies whole warp-wide slices.
// Warp-per-(row, column chunk): the row's (col, val) pairs are fetched once per warp into
// registers and broadcast with shuffles; neighbour slices are read with 128-bit loads (4 fp32
// or 8 bf16 per lane), 4 of them in flight; fp32 accumulation in CSR order (deterministic).
// Element type per launch: fp32 (parity path, backward adjoint) or bf16 (tensor-core path's
// forward diffusion blocks, which are the GEMM A operands).
#include <cuda_bf16.h>

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

template <typename T, int V>
struct Lane;
template <>
struct Lane<float, 4> {
  static __device__ __forceinline__ void load(const float *p, float *v) {
    const float4 a = __ldg(reinterpret_cast<const float4 *>(p));
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w;
  }
  static __device__ __forceinline__ void load_plain(const float *p, float *v) {
    const float4 a = *reinterpret_cast<const float4 *>(p);
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w;
  }
  static __device__ __forceinline__ void store(float *p, const float *v) {
    *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <>
struct Lane<float, 1> {
  static __device__ __forceinline__ void load(const float *p, float *v) { v[0] = __ldg(p); }
  static __device__ __forceinline__ void load_plain(const float *p, float *v) { v[0] = *p; }
  static __device__ __forceinline__ void store(float *p, const float *v) { *p = v[0]; }
};
template <>
struct Lane<__nv_bfloat16, 8> {
  static __device__ __forceinline__ void unpack(const uint4 &a, float *v) {
    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&a);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x, v[2 * i + 1] = f.y;
    }
  }
  static __device__ __forceinline__ void load(const __nv_bfloat16 *p, float *v) {
    unpack(__ldg(reinterpret_cast<const uint4 *>(p)), v);
  }
  static __device__ __forceinline__ void load_plain(const __nv_bfloat16 *p, float *v) {
    unpack(*reinterpret_cast<const uint4 *>(p), v);
  }
  static __device__ __forceinline__ void store(__nv_bfloat16 *p, const float *v) {
    uint4 a;
    __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&a);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4 *>(p) = a;
  }
};

template <typename T, int VEC>
__global__ void __launch_bounds__(256) k_spmm(const __grid_constant__ SpmmParams p) {
  using L = Lane<T, VEC>;
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

  float acc[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) acc[i] = 0.f;
  for (int t = 0; t < jb.nterms; ++t) {
    const int32_t beg = jb.rowptr[t][n], end = jb.rowptr[t][n + 1];
    const T *X = reinterpret_cast<const T *>(jb.X[t]) + goff;
    for (int32_t e0 = beg; e0 < end; e0 += 32) {
      const int cnt = min(32, end - e0);
      int32_t mycol = 0;
      float myval = 0.f;
      if (lane < cnt) mycol = __ldg(jb.col[t] + e0 + lane), myval = __ldg(jb.val[t] + e0 + lane);
      int e = 0;
      for (; e + 4 <= cnt; e += 4) {
        float xv[4][VEC], vv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = __shfl_sync(0xffffffffu, mycol, e + u);
          vv[u] = __shfl_sync(0xffffffffu, myval, e + u);
          if (active) L::load(X + int64_t(c) * jb.W + col0, xv[u]);
        }
        if (active) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int i = 0; i < VEC; ++i) acc[i] = fmaf(vv[u], xv[u][i], acc[i]);
        }
      }
      for (; e < cnt; ++e) {
        const int c = __shfl_sync(0xffffffffu, mycol, e);
        const float v = __shfl_sync(0xffffffffu, myval, e);
        if (active) {
          float xv[VEC];
          L::load(X + int64_t(c) * jb.W + col0, xv);
#pragma unroll
          for (int i = 0; i < VEC; ++i) acc[i] = fmaf(v, xv[i], acc[i]);
        }
      }
    }
  }
  if (!active) return;
  const int64_t o = goff + int64_t(n) * jb.W + col0;
  float tmp[VEC];
  if (jb.add) {
    L::load_plain(reinterpret_cast<const T *>(jb.add) + o, tmp);
#pragma unroll
    for (int i = 0; i < VEC; ++i) acc[i] += tmp[i];
  }
  T *Y = reinterpret_cast<T *>(jb.Y) + o;
  if (jb.accumulate) {
    L::load_plain(Y, tmp);
#pragma unroll
    for (int i = 0; i < VEC; ++i) acc[i] += tmp[i];
  }
  L::store(Y, acc);
}

}  // namespace

cudaError_t launch_spmm(SpmmJob *jobs, int njobs, int N, cudaStream_t s) {
  if (njobs <= 0) return cudaSuccess;
  if (njobs > kMaxSpmmJobs) return cudaErrorInvalidValue;
  const bool bf = jobs[0].bf16 != 0;
  auto al = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  bool vec = true;
  for (int i = 0; i < njobs; ++i) {
    const SpmmJob &j = jobs[i];
    if ((j.bf16 != 0) != bf) return cudaErrorInvalidValue;
    const int w = bf ? 8 : 4;
    vec = vec && j.W % w == 0 && j.gstride % w == 0 && al(j.Y) && (!j.add || al(j.add)) &&
          (j.nterms < 1 || al(j.X[0])) && (j.nterms < 2 || al(j.X[1]));
  }
  if (bf && !vec) return cudaErrorInvalidValue;  // bf16 path needs 16-byte lanes
  const int vw = bf ? 256 : (vec ? 128 : 32);
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
  const double es = bf ? 2.0 : 4.0;
  double bytes = 0.0, flops = 0.0;
  for (int i = 0; i < njobs; ++i) {
    const SpmmJob &j = jobs[i];
    const double nw = double(N) * double(j.W) * es * j.G;
    bytes += nw * (1 + j.nterms + (j.add ? 1 : 0) + (j.accumulate ? 1 : 0));
    for (int t = 0; t < j.nterms; ++t) {
      bytes += (double(j.nnz[t]) * 8.0 + double(N + 1) * 4.0) * j.G;
      flops += 2.0 * double(j.nnz[t]) * double(j.W) * j.G;
    }
  }
  ProfScope prof(kProfSpmm, s, bytes, flops);
  const unsigned blocks = unsigned(ceil_div(w, 8));
  if (bf)
    k_spmm<__nv_bfloat16, 8><<<blocks, 256, 0, s>>>(p);
  else if (vec)
    k_spmm<float, 4><<<blocks, 256, 0, s>>>(p);
  else
    k_spmm<float, 1><<<blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace pgti
