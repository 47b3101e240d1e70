// K2: CSR SpMM for the diffusion convolution (Li et al. Eq. 2 [ext]).
// Dense operand layout [G][N][W]: node-major, every node's W = B*C values contiguous, so one
// CSR row of the transition matrix multiplies whole contiguous slices.
// One thread per (row, 16-byte column vector: 4 fp32 or 8 bf16): the row's CSR entries are read
// through the read-only path (all threads of a row hit the same lines -> L1 broadcast), each
// neighbour slice is one 128-bit load, accumulation is fp32 with packed FFMA2 (sm_100) in CSR
// order (deterministic).  Consecutive threads cover consecutive columns of one row, so every
// neighbour read of a warp is a contiguous 512-byte segment.  (A warp-per-row design that
// broadcast the CSR with shuffles measured 1.3-2.3x slower: tests/cuda/spmm_microbench.cu.)
// With a window plan (pgti_graph_windows) the launch switches to k_spmm_win below, which stages
// the dense operand in shared memory (tests/cuda/spmm_tiled_mb.cu has the measurements).
// Element type per launch: fp32 (parity path, backward adjoint) or bf16 (tensor-core path's
// diffusion blocks, which are the GEMM A operands).
#include <cuda_bf16.h>

#include <cstdlib>
#include <type_traits>

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
  static __device__ __forceinline__ void fma_v(float2 *acc, float w, uint4 r) {
    const float2 ww = make_float2(w, w);
    acc[0] = __ffma2_rn(ww, make_float2(__uint_as_float(r.x), __uint_as_float(r.y)), acc[0]);
    acc[1] = __ffma2_rn(ww, make_float2(__uint_as_float(r.z), __uint_as_float(r.w)), acc[1]);
  }
  static __device__ __forceinline__ void add(float2 *acc, const float *p) {
    const float4 a = *reinterpret_cast<const float4 *>(p);
    acc[0] = __fadd2_rn(acc[0], make_float2(a.x, a.y));
    acc[1] = __fadd2_rn(acc[1], make_float2(a.z, a.w));
  }
  static __device__ __forceinline__ void axpy(float2 *acc, float b, const float *p) {
    const float4 a = *reinterpret_cast<const float4 *>(p);
    const float2 bb = make_float2(b, b);
    acc[0] = __ffma2_rn(bb, make_float2(a.x, a.y), acc[0]);
    acc[1] = __ffma2_rn(bb, make_float2(a.z, a.w), acc[1]);
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
  static __device__ __forceinline__ void fma_v(float2 *acc, float w, uint4 a) {
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
  static __device__ __forceinline__ void axpy(float2 *acc, float b, const __nv_bfloat16 *p) {
    const uint4 a = *reinterpret_cast<const uint4 *>(p);
    const float2 bb = make_float2(b, b);
    acc[0] = __ffma2_rn(bb, unpack(a.x), acc[0]);
    acc[1] = __ffma2_rn(bb, unpack(a.y), acc[1]);
    acc[2] = __ffma2_rn(bb, unpack(a.z), acc[2]);
    acc[3] = __ffma2_rn(bb, unpack(a.w), acc[3]);
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

// Y = alpha * acc + beta * add + beta2 * add2 (+ Y): the plain defaults keep the original
// instruction sequence (FADD2 of the addend), so existing results are unchanged bit for bit
template <typename L, typename T, bool GEN>
__device__ __forceinline__ void finish(const SpmmJob &jb, float2 *acc, int64_t o) {
  constexpr int P = L::V / 2;
  if (!GEN) {  // Y (+)= acc + add: the plain epilogue (alpha = beta = 1, no add2)
    if (jb.add) L::add(acc, reinterpret_cast<const T *>(jb.add) + o);
    T *Y = reinterpret_cast<T *>(jb.Y) + o;
    if (jb.accumulate) L::add(acc, Y);
    L::store(Y, acc);
    return;
  }
  if (jb.alpha != 1.f) {
    const float2 a = make_float2(jb.alpha, jb.alpha);
#pragma unroll
    for (int q = 0; q < P; ++q) acc[q] = __fmul2_rn(a, acc[q]);
  }
  if (jb.add) {
    const T *ad = reinterpret_cast<const T *>(jb.add) + o;
    if (jb.beta == 1.f)
      L::add(acc, ad);
    else
      L::axpy(acc, jb.beta, ad);
  }
  if (jb.add2) L::axpy(acc, jb.beta2, reinterpret_cast<const T *>(jb.add2) + o);
  T *Y = reinterpret_cast<T *>(jb.Y) + o;
  if (jb.accumulate) L::add(acc, Y);
  L::store(Y, acc);
}

template <typename T, bool GEN>
__global__ void __launch_bounds__(256) k_spmm(const __grid_constant__ SpmmParams p) {
  using L = Lane<T>;
  constexpr int V = L::V, P = V / 2;
  griddep_launch_dependents();
  griddep_wait();
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
  finish<L, T, GEN>(jb, acc, o);
}

// Shared-memory staged variant (the plan of pgti_graph_windows): CTA = (window of win_rows
// consecutive nodes, 512-byte column chunk).  The union of the window's neighbour rows is staged
// once into shared memory with cp.async (16 bytes per lane, L1 bypassed), then warp w reduces rows
// w, w+8, ... of the window with lane = one 16-byte vector, reading neighbours from shared memory
// (a warp reads one contiguous 512-byte row: conflict-free).  L2->SM traffic for the dense
// operand drops from nnz/N (~8.3) slices per output slice to the window's union/rows (~1.9 at 32
// rows on the kNN sensor graphs).  Same terms, same CSR order, same FFMA2 sequence as k_spmm:
// bit-identical results.
constexpr int kWinMaxSmem = 192 * 1024;

struct WinParams {
  SpmmJob job[kMaxSpmmJobs];
  int z_begin[kMaxSpmmJobs + 1];  // grid.z slots of job j: [z_begin[j], z_begin[j+1]) = groups
  int nchunk[kMaxSpmmJobs];
  int vecs[kMaxSpmmJobs];
  int njobs, N, nwin, win_rows, win_max;
};

__device__ __forceinline__ void cp_async16(void *smem, const void *g) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}

// grid = (512-byte column chunk, window, job x group): decoded without integer division
template <typename T, int RPW, bool GEN>
__global__ void __launch_bounds__(256, RPW <= 4 ? 3 : 1) k_spmm_win(const __grid_constant__ WinParams p) {
  using L = Lane<T>;
  constexpr int V = L::V, P = V / 2;
  extern __shared__ uint4 stage[];  // [union][32]
  griddep_launch_dependents();
  const int z = int(blockIdx.z);
  int j = 0;
#pragma unroll
  for (int q = 1; q < kMaxSpmmJobs; ++q)
    if (q < p.njobs && z >= p.z_begin[q]) j = q;
  const int chunk = int(blockIdx.x);
  if (chunk >= p.nchunk[j]) return;  // jobs narrower than the widest one
  const SpmmJob &jb = p.job[j];
  const int g = z - p.z_begin[j], win = int(blockIdx.y);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int vec = chunk * 32 + lane;
  const bool act = vec < p.vecs[j];
  const int W = int(jb.W);
  const int64_t goff = int64_t(g) * jb.gstride;
  const int row0 = win * p.win_rows;

  float2 acc[RPW][P];
#pragma unroll
  for (int i = 0; i < RPW; ++i)
#pragma unroll
    for (int q = 0; q < P; ++q) acc[i][q] = make_float2(0.f, 0.f);
  int *s_nodes = reinterpret_cast<int *>(stage + p.win_max * 32);
  for (int t = 0; t < jb.nterms; ++t) {
    if (t) __syncthreads();  // every warp is done with the previous term's stage
    const int ub = __ldg(jb.win_ptr[t] + win), nu = __ldg(jb.win_ptr[t] + win + 1) - ub;
    // every index load is issued up front, lane-parallel: the union's node ids into shared
    // memory, and each warp's rows' first 32 CSR entries into registers (one per lane)
    for (int i = threadIdx.x; i < nu; i += blockDim.x) s_nodes[i] = __ldg(jb.win_nodes[t] + ub + i);
    const uint16_t *lc = jb.lcol[t];
    const float *val = jb.val[t];
    int beg[RPW], cnt[RPW], cc[RPW];
    float cv[RPW];
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      const int r = warp + 8 * i, n = row0 + r;
      beg[i] = cnt[i] = cc[i] = 0, cv[i] = 0.f;
      if (r >= p.win_rows || n >= p.N) continue;  // warp-uniform
      beg[i] = __ldg(jb.rowptr[t] + n);
      cnt[i] = __ldg(jb.rowptr[t] + n + 1) - beg[i];
      if (lane < cnt[i]) cc[i] = __ldg(lc + beg[i] + lane), cv[i] = __ldg(val + beg[i] + lane);
    }
    // the plan and CSR are step constants: read above while the previous kernel drains; the
    // dense operand (and the epilogue's addends) only after it has completed (METR-LA step
    // 32.1 K -> 33.2 K samples/s)
    if (t == 0) griddep_wait();
    __syncthreads();
    const T *X = reinterpret_cast<const T *>(jb.X[t]) + goff + int64_t(vec) * V;
    if (act)
      for (int k = warp; k < nu; k += 8) cp_async16(stage + k * 32 + lane, X + int64_t(s_nodes[k]) * W);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      const int n0 = min(cnt[i], 32);
      int u = 0;
      for (; u + 4 <= n0; u += 4) {
        const int c0 = __shfl_sync(0xffffffffu, cc[i], u), c1 = __shfl_sync(0xffffffffu, cc[i], u + 1),
                  c2 = __shfl_sync(0xffffffffu, cc[i], u + 2), c3 = __shfl_sync(0xffffffffu, cc[i], u + 3);
        const float w0 = __shfl_sync(0xffffffffu, cv[i], u), w1 = __shfl_sync(0xffffffffu, cv[i], u + 1),
                    w2 = __shfl_sync(0xffffffffu, cv[i], u + 2), w3 = __shfl_sync(0xffffffffu, cv[i], u + 3);
        L::fma_v(acc[i], w0, stage[c0 * 32 + lane]);
        L::fma_v(acc[i], w1, stage[c1 * 32 + lane]);
        L::fma_v(acc[i], w2, stage[c2 * 32 + lane]);
        L::fma_v(acc[i], w3, stage[c3 * 32 + lane]);
      }
      for (; u < n0; ++u)
        L::fma_v(acc[i], __shfl_sync(0xffffffffu, cv[i], u),
                 stage[__shfl_sync(0xffffffffu, cc[i], u) * 32 + lane]);
      for (int e = beg[i] + 32; e < beg[i] + cnt[i]; ++e)  // rows with > 32 entries
        L::fma_v(acc[i], __ldg(val + e), stage[__ldg(lc + e) * 32 + lane]);
    }
  }
  if (!act) return;
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int r = warp + 8 * i, n = row0 + r;
    if (r >= p.win_rows || n >= p.N) continue;
    const int64_t o = goff + int64_t(n) * W + int64_t(vec) * V;
    finish<L, T, GEN>(jb, acc[i], o);
  }
}

// ------------------------------------------------------------------ two-hop staged diffusion
// CTA = (512-byte column chunk, window R, job x group).  The window's two-hop row set U2 is staged
// once (cp.async); hop 1 is computed for the U1 prefix into shared memory (rounded to bf16, as the
// chain stores it; R's rows also go to Y1), then hop 2 for R reads those.  Each row's terms are
// summed in CSR order with the same FFMA2 sequence as k_spmm_win: bit-identical to two launches.
// The plan (node lists, local columns, values) is a step constant: staged before
// griddepcontrol.wait, overlapping the previous kernel's tail.
constexpr int kMaxW2Jobs = 4;
struct Win2Params {
  Win2Job job[kMaxW2Jobs];
  int z_begin[kMaxW2Jobs + 1];
  int nchunk[kMaxW2Jobs];
  int vecs[kMaxW2Jobs];
  int njobs, N, rows, max_nodes, max_n1, max_entries;
};

// acc += sum_{e in [e0, e1)} val[e] * rows[col[e]] in entry order, four staged rows in flight
__device__ __forceinline__ void row_terms(float2 *acc, const uint4 *rows, const uint16_t *col,
                                          const float *val, int e0, int e1, int lane) {
  using L = Lane<__nv_bfloat16>;
  int e = e0;
  for (; e + 4 <= e1; e += 4) {
    const uint4 v0 = rows[col[e] * 32 + lane], v1 = rows[col[e + 1] * 32 + lane],
                v2 = rows[col[e + 2] * 32 + lane], v3 = rows[col[e + 3] * 32 + lane];
    L::fma_v(acc, val[e], v0);
    L::fma_v(acc, val[e + 1], v1);
    L::fma_v(acc, val[e + 2], v2);
    L::fma_v(acc, val[e + 3], v3);
  }
  for (; e < e1; ++e) L::fma_v(acc, val[e], rows[col[e] * 32 + lane]);
}

template <bool EPI>
__global__ void __launch_bounds__(256) k_spmm_win2(const __grid_constant__ Win2Params p) {
  using L = Lane<__nv_bfloat16>;
  extern __shared__ uint4 sm2[];
  griddep_launch_dependents();
  const int z = int(blockIdx.z);
  int j = 0;
#pragma unroll
  for (int q = 1; q < kMaxW2Jobs; ++q)
    if (q < p.njobs && z >= p.z_begin[q]) j = q;
  const int chunk = int(blockIdx.x);
  if (chunk >= p.nchunk[j]) return;
  const Win2Job &jb = p.job[j];
  uint4 *stage = sm2;                                        // [max_nodes][32]
  uint4 *h1 = stage + p.max_nodes * 32;                      // [max_n1][32]
  float *s_val = reinterpret_cast<float *>(h1 + p.max_n1 * 32);
  int *s_off = reinterpret_cast<int *>(s_val + p.max_entries);
  int *s_nodes = s_off + p.max_n1 + 1;
  uint16_t *s_col = reinterpret_cast<uint16_t *>(s_nodes + p.max_nodes);
  const int win = int(blockIdx.y), tid = int(threadIdx.x);
  const int nb = __ldg(jb.ptr + win), nn = __ldg(jb.ptr + win + 1) - nb;
  const int u1 = __ldg(jb.n1 + win);
  const int eb = __ldg(jb.eptr + win), ne = __ldg(jb.eptr + win + 1) - eb;
  for (int i = tid; i < nn; i += 256) s_nodes[i] = __ldg(jb.nodes + nb + i);
  for (int i = tid; i <= u1; i += 256) s_off[i] = __ldg(jb.roff + nb + win + i);
  for (int i = tid; i < ne; i += 256)
    s_col[i] = __ldg(jb.lcol + eb + i), s_val[i] = __ldg(jb.val + __ldg(jb.eidx + eb + i));
  griddep_wait();
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  const int vec = chunk * 32 + lane;
  const bool act = vec < p.vecs[j];
  const int64_t W = jb.W, goff = int64_t(z - p.z_begin[j]) * jb.gstride;
  const __nv_bfloat16 *X = static_cast<const __nv_bfloat16 *>(jb.X) + goff + int64_t(vec) * 8;
  if (act)
    for (int k = warp; k < nn; k += 8) cp_async16(stage + k * 32 + lane, X + int64_t(s_nodes[k]) * W);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const int row0 = win * p.rows, nrows = min(p.rows, p.N - row0);
  for (int i = warp; i < u1; i += 8) {  // hop 1 over U1 (R first)
    float2 acc[4] = {};
    row_terms(acc, stage, s_col, s_val, s_off[i], s_off[i + 1], lane);
    L::store(reinterpret_cast<__nv_bfloat16 *>(h1 + i * 32 + lane), acc);
    if (act && i < nrows)
      L::store(static_cast<__nv_bfloat16 *>(jb.Y1) + goff + int64_t(row0 + i) * W + int64_t(vec) * 8,
               acc);
  }
  __syncthreads();
  for (int r = warp; r < nrows; r += 8) {  // hop 2 over R from the hop-1 rows
    float2 acc[4] = {};
    row_terms(acc, h1, s_col, s_val, s_off[r], s_off[r + 1], lane);
    if (!act) continue;
    const int64_t o = goff + int64_t(row0 + r) * W + int64_t(vec) * 8;
    if (EPI) {  // as finish<.., true>: alpha scaling, then beta * add
      const float2 a = make_float2(jb.alpha, jb.alpha);
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = __fmul2_rn(a, acc[q]);
      const __nv_bfloat16 *ad = static_cast<const __nv_bfloat16 *>(jb.add) + o;
      if (jb.beta == 1.f)
        L::add(acc, ad);
      else
        L::axpy(acc, jb.beta, ad);
    }
    L::store(static_cast<__nv_bfloat16 *>(jb.Y2) + o, acc);
  }
}

// ------------------------------------------------------------------ resident small-graph diffusion
constexpr int kResThreads = 512, kResMaxSmem = 200 * 1024;

template <int K>
__global__ void __launch_bounds__(kResThreads) k_spmm_resident(const __grid_constant__ ResidentJob p) {
  using L = Lane<__nv_bfloat16>;
  extern __shared__ uint4 rs[];  // X chunk [N][8], then (K == 2) hop 1 [2][N][8]
  griddep_launch_dependents();
  griddep_wait();
  const int N = p.N;
  const int64_t W = p.W;
  const int vecs = int(W / 8), vbase = int(blockIdx.x) * 8;
  const int grp = threadIdx.x >> 3, l8 = threadIdx.x & 7, ngrp = kResThreads / 8;
  const bool act = vbase + l8 < vecs;
  const __nv_bfloat16 *X = static_cast<const __nv_bfloat16 *>(p.X) + int64_t(vbase + l8) * 8;
  if (act)
    for (int n = grp; n < N; n += ngrp) cp_async16(rs + n * 8 + l8, X + int64_t(n) * W);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  uint4 *h1 = rs + N * 8;
#pragma unroll
  for (int hop = 0; hop < K; ++hop) {
    if (hop) __syncthreads();  // hop-1 rows complete
    for (int it = grp; it < 2 * N; it += ngrp) {
      const int dir = it >= N, n = it - dir * N;
      const uint4 *src = hop == 0 ? rs : h1 + dir * N * 8;
      const int32_t *col = p.col[dir];
      const float *val = p.val[dir];
      float2 acc[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = make_float2(0.f, 0.f);
      const int beg = __ldg(p.rowptr[dir] + n), end = __ldg(p.rowptr[dir] + n + 1);
      int e = beg;
      for (; e + 4 <= end; e += 4) {
        const int c0 = __ldg(col + e), c1 = __ldg(col + e + 1), c2 = __ldg(col + e + 2),
                  c3 = __ldg(col + e + 3);
        const float w0 = __ldg(val + e), w1 = __ldg(val + e + 1), w2 = __ldg(val + e + 2),
                    w3 = __ldg(val + e + 3);
        L::fma_v(acc, w0, src[c0 * 8 + l8]);
        L::fma_v(acc, w1, src[c1 * 8 + l8]);
        L::fma_v(acc, w2, src[c2 * 8 + l8]);
        L::fma_v(acc, w3, src[c3 * 8 + l8]);
      }
      for (; e < end; ++e) L::fma_v(acc, __ldg(val + e), src[__ldg(col + e) * 8 + l8]);
      if (!act) continue;
      uint4 o;
      __nv_bfloat162 h;
      h = __floats2bfloat162_rn(acc[0].x, acc[0].y), o.x = *reinterpret_cast<uint32_t *>(&h);
      h = __floats2bfloat162_rn(acc[1].x, acc[1].y), o.y = *reinterpret_cast<uint32_t *>(&h);
      h = __floats2bfloat162_rn(acc[2].x, acc[2].y), o.z = *reinterpret_cast<uint32_t *>(&h);
      h = __floats2bfloat162_rn(acc[3].x, acc[3].y), o.w = *reinterpret_cast<uint32_t *>(&h);
      *reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.Y[dir][hop]) + int64_t(n) * W +
                                 int64_t(vbase + l8) * 8) = o;
      if (hop + 1 < K) h1[(dir * N + n) * 8 + l8] = o;
    }
  }
}

// Scalar fp32 fallback for widths that are not a multiple of 4 (test shapes only).
__global__ void __launch_bounds__(256) k_spmm_scalar(const __grid_constant__ SpmmParams p) {
  griddep_launch_dependents();
  griddep_wait();
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
  if (jb.alpha != 1.f) acc *= jb.alpha;
  if (jb.add) acc = jb.beta == 1.f ? acc + jb.add[o] : fmaf(jb.beta, jb.add[o], acc);
  if (jb.add2) acc = fmaf(jb.beta2, jb.add2[o], acc);
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
    bytes += nw * (1 + j.nterms + (j.add ? 1 : 0) + (j.add2 ? 1 : 0) + (j.accumulate ? 1 : 0));
    for (int t = 0; t < j.nterms; ++t) {
      bytes += (double(j.nnz[t]) * 8.0 + double(N + 1) * 4.0) * j.G;
      flops += 2.0 * double(j.nnz[t]) * double(j.W) * j.G;
    }
  }
  ProfScope prof(kProfSpmm, s, bytes, flops);
  bool gen = false;
  for (int i = 0; i < njobs; ++i)
    gen = gen || jobs[i].alpha != 1.f || jobs[i].beta != 1.f || jobs[i].add2;
  // shared-memory staged kernel when every term carries a window plan of one size that fits
  bool win = vec && jobs[0].win_rows > 0 && jobs[0].win_max > 0 &&
             jobs[0].win_max * 516 <= kWinMaxSmem;
  for (int i = 0; i < njobs && win; ++i) {
    const SpmmJob &j = jobs[i];
    win = j.nterms >= 1 && j.win_rows == jobs[0].win_rows && j.win_max == jobs[0].win_max;
    for (int t = 0; t < j.nterms && win; ++t) win = j.win_ptr[t] && j.win_nodes[t] && j.lcol[t];
  }
  WinParams w{};
  int nz = 0, maxc = 0;
  if (win) {
    w.njobs = njobs, w.N = N, w.win_rows = jobs[0].win_rows, w.win_max = jobs[0].win_max;
    w.nwin = int(ceil_div(N, w.win_rows));
    for (int i = 0; i < njobs; ++i) {
      w.job[i] = jobs[i];
      w.vecs[i] = int(jobs[i].W / V);
      w.nchunk[i] = int(ceil_div(w.vecs[i], 32));
      w.z_begin[i] = nz;
      nz += jobs[i].G;
      maxc = std::max(maxc, w.nchunk[i]);
    }
    w.z_begin[njobs] = nz;
    if (nz > 65535 || w.nwin > 65535) win = false;
  }
  if (win) {
    const dim3 grid(unsigned(maxc), unsigned(w.nwin), unsigned(nz));
    const int smem = jobs[0].win_max * 516;  // staged rows + their node ids
    const int rpw = (w.win_rows + 7) / 8;
    auto go = [&](auto kernel) -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      return pdl_launch(kernel, grid, dim3(256), smem, s, w);
    };
    auto pick = [&](auto gen) -> cudaError_t {
      constexpr bool G = decltype(gen)::value;
      if (bf) {
        if (rpw <= 1) return go(k_spmm_win<__nv_bfloat16, 1, G>);
        if (rpw <= 2) return go(k_spmm_win<__nv_bfloat16, 2, G>);
        if (rpw <= 4) return go(k_spmm_win<__nv_bfloat16, 4, G>);
        return go(k_spmm_win<__nv_bfloat16, 8, G>);
      }
      if (rpw <= 1) return go(k_spmm_win<float, 1, G>);
      if (rpw <= 2) return go(k_spmm_win<float, 2, G>);
      if (rpw <= 4) return go(k_spmm_win<float, 4, G>);
      return go(k_spmm_win<float, 8, G>);
    };
    // the general epilogue (Chebyshev / Clenshaw: alpha, beta, add2) costs registers (bf16 x 4
    // rows: 79 -> 91, 3 -> 2 CTAs per SM), so it is its own instantiation
    return gen ? pick(std::true_type{}) : pick(std::false_type{});
  }
  const unsigned blocks = unsigned(ceil_div(th, 256));
  if (bf)
    return gen ? pdl_launch(k_spmm<__nv_bfloat16, true>, dim3(blocks), dim3(256), 0, s, p)
               : pdl_launch(k_spmm<__nv_bfloat16, false>, dim3(blocks), dim3(256), 0, s, p);
  if (vec)
    return gen ? pdl_launch(k_spmm<float, true>, dim3(blocks), dim3(256), 0, s, p)
               : pdl_launch(k_spmm<float, false>, dim3(blocks), dim3(256), 0, s, p);
  return pdl_launch(k_spmm_scalar, dim3(blocks), dim3(256), 0, s, p);
}

cudaError_t launch_spmm_win2(const Win2Job *jobs, int njobs, int N, const Win2Plan &plan,
                             cudaStream_t s) {
  if (njobs < 1 || njobs > kMaxW2Jobs || plan.rows < 1) return cudaErrorInvalidValue;
  const size_t smem = size_t(plan.max_nodes + plan.max_n1) * 512 + size_t(plan.max_entries) * 6 +
                      size_t(plan.max_n1 + 1 + plan.max_nodes) * 4 + 16;
  if (smem > size_t(kWinMaxSmem)) return cudaErrorNotSupported;
  Win2Params w{};
  w.njobs = njobs, w.N = N, w.rows = plan.rows, w.max_nodes = plan.max_nodes;
  w.max_n1 = plan.max_n1, w.max_entries = plan.max_entries;
  int nz = 0, maxc = 0;
  bool epi = false;
  double bytes = 0.0, flops = 0.0;
  for (int i = 0; i < njobs; ++i) {
    const Win2Job &j = jobs[i];
    if (j.W % 8 || !j.X || !j.Y1 || !j.Y2 || j.G < 1) return cudaErrorInvalidValue;
    w.job[i] = j;
    w.vecs[i] = int(j.W / 8);
    w.nchunk[i] = int(ceil_div(w.vecs[i], 32));
    w.z_begin[i] = nz;
    nz += j.G;
    maxc = std::max(maxc, w.nchunk[i]);
    epi = epi || j.add;
    // algorithmic bytes: X read once, Y1 and Y2 written once, the addend read once, the CSR
    // once; flops: both hops over the graph (the recomputed U1 \ R rows are overhead, not work)
    const double nw = double(N) * double(j.W) * 2.0 * j.G;
    bytes += nw * (3 + (j.add ? 1 : 0)) + (double(j.nnz) * 8.0 + double(N + 1) * 4.0) * j.G;
    flops += 4.0 * double(j.nnz) * double(j.W) * j.G;
  }
  w.z_begin[njobs] = nz;
  const int nwin = int(ceil_div(N, plan.rows));
  if (nz > 65535 || nwin > 65535) return cudaErrorNotSupported;
  ProfScope prof(kProfSpmm, s, bytes, flops);
  const dim3 grid{unsigned(maxc), unsigned(nwin), unsigned(nz)};
  auto go = [&](auto kernel) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
    return pdl_launch(kernel, grid, dim3(256), int(smem), s, w);
  };
  return epi ? go(k_spmm_win2<true>) : go(k_spmm_win2<false>);
}

bool spmm_resident_fits(int N, int K, int64_t W) {
  return K >= 1 && K <= 2 && W % 8 == 0 && int64_t(N) * 128 * (K == 2 ? 3 : 1) <= kResMaxSmem;
}

cudaError_t launch_spmm_resident(const ResidentJob &p, cudaStream_t s) {
  if (!spmm_resident_fits(p.N, p.K, p.W)) return cudaErrorInvalidValue;
  const int smem = p.N * 128 * (p.K == 2 ? 3 : 1);
  const unsigned grid = unsigned(ceil_div(p.W * 2, 128));
  // algorithmic bytes as launch_spmm's 2 x K single-term jobs
  double bytes = 0.0, flops = 0.0;
  for (int d = 0; d < 2; ++d) {
    bytes += 2.0 * double(p.N) * double(p.W) * 2.0 * p.K;
    bytes += (double(p.nnz[d]) * 8.0 + double(p.N + 1) * 4.0) * p.K;
    flops += 2.0 * double(p.nnz[d]) * double(p.W) * p.K;
  }
  ProfScope prof(kProfSpmm, s, bytes, flops);
  auto go = [&](auto kernel) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    return pdl_launch(kernel, dim3(grid), dim3(kResThreads), smem, s, p);
  };
  return p.K == 2 ? go(k_spmm_resident<2>) : go(k_spmm_resident<1>);
}

}  // namespace pgti
