// K2: CSR SpMM for the diffusion convolution (Li et al. Eq. 2 [ext]).
// Dense operand layout [G][N][W]: node-major, every node's W = B*C values contiguous, so one
// CSR row of the transition matrix multiplies whole warp-wide slices.
// One warp per (row, run of CPW column chunks): the row's (col, val) pairs are loaded once
// (lane e holds entry e), broadcast with shuffles, and reused for every chunk of the run;
// neighbour slices are read with 128-bit loads (4 fp32 or 8 bf16 per lane), 4 in flight, and
// accumulated in fp32 with packed FFMA2 (sm_100) in CSR order (deterministic).
// Element type per launch: fp32 (parity path, backward adjoint) or bf16 (tensor-core path's
// diffusion blocks, which are the GEMM A operands).
#include <cuda_bf16.h>

#include "kernels.cuh"
#include "profile.cuh"

namespace pgti {
namespace {

struct SpmmParams {
  SpmmJob job[kMaxSpmmJobs];
  int warp_begin[kMaxSpmmJobs + 1];
  int runs[kMaxSpmmJobs];   // runs (of CPW chunks) per row
  int chunks[kMaxSpmmJobs];
  int njobs;
  int N;
};

constexpr int kCPW = 1;   // chunks per warp run
constexpr int kGrp = 4;   // neighbour loads in flight per lane

template <typename T>
struct Lane;
template <>
struct Lane<float> {
  static constexpr int V = 4;
  using Raw = float4;
  static __device__ __forceinline__ Raw ld_raw(const float *p) {
    return __ldg(reinterpret_cast<const float4 *>(p));
  }
  static __device__ __forceinline__ void fma_raw(float2 *acc, float w, const Raw &a) {
    const float2 ww = make_float2(w, w);
    acc[0] = __ffma2_rn(ww, make_float2(a.x, a.y), acc[0]);
    acc[1] = __ffma2_rn(ww, make_float2(a.z, a.w), acc[1]);
  }
  static __device__ __forceinline__ void load(const float *p, float2 *v) {
    const float4 a = __ldg(reinterpret_cast<const float4 *>(p));
    v[0] = make_float2(a.x, a.y), v[1] = make_float2(a.z, a.w);
  }
  static __device__ __forceinline__ void load_plain(const float *p, float2 *v) {
    const float4 a = *reinterpret_cast<const float4 *>(p);
    v[0] = make_float2(a.x, a.y), v[1] = make_float2(a.z, a.w);
  }
  static __device__ __forceinline__ void store(float *p, const float2 *v) {
    *reinterpret_cast<float4 *>(p) = make_float4(v[0].x, v[0].y, v[1].x, v[1].y);
  }
};
template <>
struct Lane<__nv_bfloat16> {
  static constexpr int V = 8;
  static __device__ __forceinline__ float2 unpack(uint32_t w) {
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
  }
  using Raw = uint4;
  static __device__ __forceinline__ Raw ld_raw(const __nv_bfloat16 *p) {
    return __ldg(reinterpret_cast<const uint4 *>(p));
  }
  static __device__ __forceinline__ void fma_raw(float2 *acc, float w, const Raw &a) {
    const float2 ww = make_float2(w, w);
    acc[0] = __ffma2_rn(ww, unpack(a.x), acc[0]);
    acc[1] = __ffma2_rn(ww, unpack(a.y), acc[1]);
    acc[2] = __ffma2_rn(ww, unpack(a.z), acc[2]);
    acc[3] = __ffma2_rn(ww, unpack(a.w), acc[3]);
  }
  static __device__ __forceinline__ void load(const __nv_bfloat16 *p, float2 *v) {
    const uint4 a = __ldg(reinterpret_cast<const uint4 *>(p));
    v[0] = unpack(a.x), v[1] = unpack(a.y), v[2] = unpack(a.z), v[3] = unpack(a.w);
  }
  static __device__ __forceinline__ void load_plain(const __nv_bfloat16 *p, float2 *v) {
    const uint4 a = *reinterpret_cast<const uint4 *>(p);
    v[0] = unpack(a.x), v[1] = unpack(a.y), v[2] = unpack(a.z), v[3] = unpack(a.w);
  }
  static __device__ __forceinline__ void store(__nv_bfloat16 *p, const float2 *v) {
    uint4 a;
    __nv_bfloat162 h;
    h = __floats2bfloat162_rn(v[0].x, v[0].y), a.x = *reinterpret_cast<uint32_t *>(&h);
    h = __floats2bfloat162_rn(v[1].x, v[1].y), a.y = *reinterpret_cast<uint32_t *>(&h);
    h = __floats2bfloat162_rn(v[2].x, v[2].y), a.z = *reinterpret_cast<uint32_t *>(&h);
    h = __floats2bfloat162_rn(v[3].x, v[3].y), a.w = *reinterpret_cast<uint32_t *>(&h);
    *reinterpret_cast<uint4 *>(p) = a;
  }
};

template <typename T>
__global__ void __launch_bounds__(256, 4) k_spmm(const __grid_constant__ SpmmParams p) {
  using L = Lane<T>;
  constexpr int V = L::V, P = V / 2;
  const int wid = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (wid >= p.warp_begin[p.njobs]) return;
  int j = 0;
#pragma unroll
  for (int q = 1; q < kMaxSpmmJobs; ++q)
    if (q < p.njobs && wid >= p.warp_begin[q]) j = q;
  const SpmmJob &jb = p.job[j];
  const int runs = p.runs[j], chunks = p.chunks[j];
  int rem = wid - p.warp_begin[j];
  const int per_group = p.N * runs;
  const int g = rem / per_group;
  rem -= g * per_group;
  const int n = rem / runs;
  const int run = rem - n * runs;
  const int W = int(jb.W);
  const int64_t orow = int64_t(g) * jb.gstride + int64_t(n) * W;
  for (int c = run * kCPW; c < min(chunks, run * kCPW + kCPW); ++c) {
    const int col0 = c * 32 * V + lane * V;
    const bool active = col0 < W;
    float2 acc[P];
#pragma unroll
    for (int i = 0; i < P; ++i) acc[i] = make_float2(0.f, 0.f);
    for (int t = 0; t < jb.nterms; ++t) {
      const T *base = reinterpret_cast<const T *>(jb.X[t]) + int64_t(g) * jb.gstride + col0;
      const int beg = __ldg(jb.rowptr[t] + n), cnt = __ldg(jb.rowptr[t] + n + 1) - beg;
      for (int e0 = 0; e0 < cnt; e0 += 32) {
        // lane e holds CSR entry e0 + e of the row; broadcast with shuffles
        const int ce = min(32, cnt - e0);
        int cc = 0;
        float vv = 0.f;
        if (lane < ce) cc = __ldg(jb.col[t] + beg + e0 + lane), vv = __ldg(jb.val[t] + beg + e0 + lane);
        // all (up to kGrp) neighbour slices of the group in flight before any FMA
        for (int e = 0; e < ce; e += kGrp) {
          typename L::Raw xr[kGrp];
          float w[kGrp];
#pragma unroll
          for (int u = 0; u < kGrp; ++u) {
            const int col = __shfl_sync(0xffffffffu, cc, (e + u) & 31);
            w[u] = __shfl_sync(0xffffffffu, vv, (e + u) & 31);
            if (active && e + u < ce) xr[u] = L::ld_raw(base + col * W);
          }
          if (active) {
#pragma unroll
            for (int u = 0; u < kGrp; ++u)
              if (e + u < ce) L::fma_raw(acc, w[u], xr[u]);
          }
        }
      }
    }
    if (!active) continue;
    float2 tmp[P];
    if (jb.add) {
      L::load_plain(reinterpret_cast<const T *>(jb.add) + orow + col0, tmp);
#pragma unroll
      for (int i = 0; i < P; ++i) acc[i] = __fadd2_rn(acc[i], tmp[i]);
    }
    T *Y = reinterpret_cast<T *>(jb.Y) + orow + col0;
    if (jb.accumulate) {
      L::load_plain(Y, tmp);
#pragma unroll
      for (int i = 0; i < P; ++i) acc[i] = __fadd2_rn(acc[i], tmp[i]);
    }
    L::store(Y, acc);
  }
}

// Scalar fp32 fallback for widths that are not a multiple of 4 (test shapes only).
__global__ void __launch_bounds__(256) k_spmm_scalar(const __grid_constant__ SpmmParams p) {
  const int wid = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (wid >= p.warp_begin[p.njobs]) return;
  int j = 0;
  for (int q = 1; q < p.njobs; ++q)
    if (wid >= p.warp_begin[q]) j = q;
  const SpmmJob &jb = p.job[j];
  const int runs = p.runs[j];
  int rem = wid - p.warp_begin[j];
  const int g = rem / (p.N * runs);
  rem -= g * p.N * runs;
  const int n = rem / runs, run = rem - (rem / runs) * runs;
  const int W = int(jb.W);
  const int64_t orow = int64_t(g) * jb.gstride + int64_t(n) * W;
  for (int col = run * 32 + lane; col < W; col += runs * 32) {
    float acc = 0.f;
    for (int t = 0; t < jb.nterms; ++t) {
      const float *X = jb.X[t] + int64_t(g) * jb.gstride;
      for (int e = jb.rowptr[t][n]; e < jb.rowptr[t][n + 1]; ++e)
        acc = fmaf(jb.val[t][e], X[int64_t(jb.col[t][e]) * W + col], acc);
    }
    if (jb.add) acc += jb.add[orow + col];
    if (jb.accumulate) acc += jb.Y[orow + col];
    jb.Y[orow + col] = acc;
  }
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
    if (int64_t(N) * j.W >= (int64_t(1) << 31)) return cudaErrorInvalidValue;  // 32-bit offsets
    const int w = bf ? 8 : 4;
    vec = vec && j.W % w == 0 && j.gstride % w == 0 && al(j.Y) && (!j.add || al(j.add)) &&
          (j.nterms < 1 || al(j.X[0])) && (j.nterms < 2 || al(j.X[1]));
  }
  if (bf && !vec) return cudaErrorInvalidValue;  // bf16 path needs 16-byte lanes
  const int vw = bf ? 256 : 128;
  SpmmParams p{};
  int64_t w = 0;
  for (int i = 0; i < njobs; ++i) {
    p.job[i] = jobs[i];
    if (p.job[i].nterms < 2) p.job[i].X[1] = p.job[i].X[0];
    p.chunks[i] = int(ceil_div(jobs[i].W, vw));
    p.runs[i] = vec ? int(ceil_div(p.chunks[i], kCPW)) : 1;
    p.warp_begin[i] = int(w);
    w += int64_t(jobs[i].G) * N * p.runs[i];
  }
  if (w >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
  p.warp_begin[njobs] = int(w);
  p.njobs = njobs;
  p.N = N;
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
    k_spmm<__nv_bfloat16><<<blocks, 256, 0, s>>>(p);
  else if (vec)
    k_spmm<float><<<blocks, 256, 0, s>>>(p);
  else
    k_spmm_scalar<<<blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace pgti
