// K2: CSR SpMM for the diffusion convolution (Li et al. Eq. 2 [ext]).
// Dense operand layout [G][N][W]: node-major, every node's W = B*C values contiguous, so one
// CSR row of the transition matrix multiplies whole contiguous slices.
// One thread per (row, 16-byte column vector: 4 fp32 or 8 bf16): the row's CSR entries are read
// through the read-only path (all threads of a row hit the same lines -> L1 broadcast), each
// neighbour slice is one 128-bit load, accumulation is fp32 with packed FFMA2 (sm_100) in CSR
// order (deterministic).  Consecutive threads cover consecutive columns of one row, so every
// neighbour read of a warp is a contiguous 512-byte segment.  (A warp-per-row design that
// broadcast the CSR with shuffles measured 1.3-2.3x slower: tests/cuda/spmm_microbench.cu.)
// Element type per launch: fp32 (parity path, backward adjoint) or bf16 (tensor-core path's
// diffusion blocks, which are the GEMM A operands).
#include <cuda_bf16.h>

#include "kernels.cuh"
#include "profile.cuh"

namespace pgti {
namespace {

struct SpmmParams {
  SpmmJob job[kMaxSpmmJobs];
  int thread_begin[kMaxSpmmJobs + 1];
  int vecs[kMaxSpmmJobs];  // 16-byte vectors per row
  int njobs;
  int N;
};

template <typename T>
struct Lane;
template <>
struct Lane<float> {
  static constexpr int V = 4;
  static __device__ __forceinline__ void fma(float2 *acc, float w, const float *p) {
    const float4 a = __ldg(reinterpret_cast<const float4 *>(p));
    const float2 ww = make_float2(w, w);
    acc[0] = __ffma2_rn(ww, make_float2(a.x, a.y), acc[0]);
    acc[1] = __ffma2_rn(ww, make_float2(a.z, a.w), acc[1]);
  }
  static __device__ __forceinline__ void add(float2 *acc, const float *p) {
    const float4 a = *reinterpret_cast<const float4 *>(p);
    acc[0] = __fadd2_rn(acc[0], make_float2(a.x, a.y));
    acc[1] = __fadd2_rn(acc[1], make_float2(a.z, a.w));
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
  static __device__ __forceinline__ void fma(float2 *acc, float w, const __nv_bfloat16 *p) {
    const uint4 a = __ldg(reinterpret_cast<const uint4 *>(p));
    const float2 ww = make_float2(w, w);
    acc[0] = __ffma2_rn(ww, unpack(a.x), acc[0]);
    acc[1] = __ffma2_rn(ww, unpack(a.y), acc[1]);
    acc[2] = __ffma2_rn(ww, unpack(a.z), acc[2]);
    acc[3] = __ffma2_rn(ww, unpack(a.w), acc[3]);
  }
  static __device__ __forceinline__ void add(float2 *acc, const __nv_bfloat16 *p) {
    const uint4 a = *reinterpret_cast<const uint4 *>(p);
    acc[0] = __fadd2_rn(acc[0], unpack(a.x));
    acc[1] = __fadd2_rn(acc[1], unpack(a.y));
    acc[2] = __fadd2_rn(acc[2], unpack(a.z));
    acc[3] = __fadd2_rn(acc[3], unpack(a.w));
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
__global__ void __launch_bounds__(256) k_spmm(const __grid_constant__ SpmmParams p) {
  using L = Lane<T>;
  constexpr int V = L::V, P = V / 2;
  const int tid = int(blockIdx.x * blockDim.x + threadIdx.x);
  if (tid >= p.thread_begin[p.njobs]) return;
  int j = 0;
#pragma unroll
  for (int q = 1; q < kMaxSpmmJobs; ++q)
    if (q < p.njobs && tid >= p.thread_begin[q]) j = q;
  const SpmmJob &jb = p.job[j];
  const int vecs = p.vecs[j];
  int rem = tid - p.thread_begin[j];
  const int per_group = p.N * vecs;
  const int g = rem / per_group;
  rem -= g * per_group;
  const int n = rem / vecs;
  const int col0 = (rem - n * vecs) * V;
  const int W = int(jb.W);
  const int64_t goff = int64_t(g) * jb.gstride;

  float2 acc[P];
#pragma unroll
  for (int i = 0; i < P; ++i) acc[i] = make_float2(0.f, 0.f);
  for (int t = 0; t < jb.nterms; ++t) {
    const T *X = reinterpret_cast<const T *>(jb.X[t]) + goff + col0;
    const int beg = __ldg(jb.rowptr[t] + n), end = __ldg(jb.rowptr[t] + n + 1);
    int e = beg;
    for (; e + 4 <= end; e += 4) {  // 4 independent neighbour loads in flight
      const int c0 = __ldg(jb.col[t] + e), c1 = __ldg(jb.col[t] + e + 1);
      const int c2 = __ldg(jb.col[t] + e + 2), c3 = __ldg(jb.col[t] + e + 3);
      const float w0 = __ldg(jb.val[t] + e), w1 = __ldg(jb.val[t] + e + 1);
      const float w2 = __ldg(jb.val[t] + e + 2), w3 = __ldg(jb.val[t] + e + 3);
      L::fma(acc, w0, X + c0 * W);
      L::fma(acc, w1, X + c1 * W);
      L::fma(acc, w2, X + c2 * W);
      L::fma(acc, w3, X + c3 * W);
    }
    for (; e < end; ++e) L::fma(acc, __ldg(jb.val[t] + e), X + __ldg(jb.col[t] + e) * W);
  }
  const int64_t o = goff + int64_t(n) * W + col0;
  if (jb.add) L::add(acc, reinterpret_cast<const T *>(jb.add) + o);
  T *Y = reinterpret_cast<T *>(jb.Y) + o;
  if (jb.accumulate) L::add(acc, Y);
  L::store(Y, acc);
}

// Scalar fp32 fallback for widths that are not a multiple of 4 (test shapes only).
__global__ void __launch_bounds__(256) k_spmm_scalar(const __grid_constant__ SpmmParams p) {
  const int tid = int(blockIdx.x * blockDim.x + threadIdx.x);
  if (tid >= p.thread_begin[p.njobs]) return;
  int j = 0;
  for (int q = 1; q < p.njobs; ++q)
    if (tid >= p.thread_begin[q]) j = q;
  const SpmmJob &jb = p.job[j];
  const int W = int(jb.W);
  int rem = tid - p.thread_begin[j];
  const int g = rem / (p.N * W);
  rem -= g * p.N * W;
  const int n = rem / W, col = rem - n * W;
  const int64_t goff = int64_t(g) * jb.gstride, o = goff + int64_t(n) * W + col;
  float acc = 0.f;
  for (int t = 0; t < jb.nterms; ++t) {
    const float *X = jb.X[t] + goff;
    for (int e = jb.rowptr[t][n]; e < jb.rowptr[t][n + 1]; ++e)
      acc = fmaf(jb.val[t][e], X[int64_t(jb.col[t][e]) * W + col], acc);
  }
  if (jb.add) acc += jb.add[o];
  if (jb.accumulate) acc += jb.Y[o];
  jb.Y[o] = acc;
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
  const int V = bf ? 8 : (vec ? 4 : 1);
  SpmmParams p{};
  int64_t th = 0;
  for (int i = 0; i < njobs; ++i) {
    p.job[i] = jobs[i];
    p.vecs[i] = int(jobs[i].W / V);
    p.thread_begin[i] = int(th);
    th += int64_t(jobs[i].G) * N * p.vecs[i];
  }
  if (th >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
  p.thread_begin[njobs] = int(th);
  p.njobs = njobs;
  p.N = N;
  if (th == 0) return cudaSuccess;
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
  const unsigned blocks = unsigned(ceil_div(th, 256));
  if (bf)
    k_spmm<__nv_bfloat16><<<blocks, 256, 0, s>>>(p);
  else if (vec)
    k_spmm<float><<<blocks, 256, 0, s>>>(p);
  else
    k_spmm_scalar<<<blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace pgti
