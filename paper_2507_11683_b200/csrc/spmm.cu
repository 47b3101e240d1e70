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
// EPI 0: Y = acc (no addend, no accumulation: every hop of the tensor-core step); 1: the plain
// Y (+)= acc + add; 2: the general form below
template <typename L, typename T, int EPI>
__device__ __forceinline__ void finish(const SpmmJob &jb, float2 *acc, int64_t o) {
  constexpr int P = L::V / 2;
  if (EPI == 0) {
    L::store(reinterpret_cast<T *>(jb.Y) + o, acc);
    return;
  }
  if (EPI == 1) {  // Y (+)= acc + add: the plain epilogue (alpha = beta = 1, no add2)
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
  finish<L, T, GEN ? 2 : 1>(jb, acc, o);
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

// grid = (column chunk of VPL x 512 bytes, window, job x group): decoded without integer
// division.  Lane l covers the 16-byte vectors l, l+32, .. (VPL of them) of the chunk, so every
// warp-wide shared-memory access is a contiguous 512-byte row segment (conflict-free) and each
// CSR entry's broadcast (one LDS.64 of (staged-row byte offset, value) from a per-warp list,
// written once per row) and address arithmetic serve VPL vectors.  Per entry and vector: one
// LDS.128 of the staged neighbour slice, the bf16 -> fp32 unpack and the FFMA2s.
constexpr int kWinEntBytes = 8 * 4 * 32 * 8;  // [warp][row slot][32] int2, RPW <= 4

template <typename T, int RPW, int VPL, int EPI>
__global__ void __launch_bounds__(256, VPL == 1 ? (RPW <= 4 ? 3 : 1) : (RPW <= 2 ? 3 : 2))
    k_spmm_win(const __grid_constant__ WinParams p) {
  using L = Lane<T>;
  constexpr int V = L::V, P = V / 2;
  constexpr int SLOTS = RPW <= 4 ? RPW : 4;  // entry lists held at once (RPW 8: two passes)
  constexpr int ROWB = 512 * VPL;            // bytes of one staged row
  extern __shared__ uint4 stage[];  // [union][32 VPL] | entries [8][SLOTS][32]
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
  const int vec0 = chunk * 32 * VPL + lane;
  const int vecs = p.vecs[j];
  const int W = int(jb.W);
  const int64_t goff = int64_t(g) * jb.gstride;
  const int row0 = win * p.win_rows;

  float2 acc[RPW][VPL][P];
#pragma unroll
  for (int i = 0; i < RPW; ++i)
#pragma unroll
    for (int v = 0; v < VPL; ++v)
#pragma unroll
      for (int q = 0; q < P; ++q) acc[i][v][q] = make_float2(0.f, 0.f);
  int2 *s_ent = reinterpret_cast<int2 *>(stage + p.win_max * 32 * VPL) + warp * (SLOTS * 32);
  const char *lane_stage = reinterpret_cast<const char *>(stage + lane);
  for (int t = 0; t < jb.nterms; ++t) {
    if (t) __syncthreads();  // every warp is done with the previous term's stage and entries
    const int ub = __ldg(jb.win_ptr[t] + win), nu = __ldg(jb.win_ptr[t] + win + 1) - ub;
    // index loads first, all independent and lane-parallel, consumed late so their latencies
    // overlap: warp w stages union rows w, w+8, .. -- lane l holds the node id of row w + 8 l
    // (rows past 8 x 32 come through the fallback loop below); and each of this warp's rows'
    // first 32 CSR entries (lane u: entry u) as (staged-row byte offset, value)
    const int my_node = warp + 8 * lane < nu ? __ldg(jb.win_nodes[t] + ub + warp + 8 * lane) : 0;
    const uint16_t *lc = jb.lcol[t];
    const float *val = jb.val[t];
    int beg[RPW], cnt[RPW];
    int2 ent[SLOTS];
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      const int r = warp + 8 * i, n = row0 + r;
      beg[i] = cnt[i] = 0;
      if (i < SLOTS) ent[i] = make_int2(0, 0);
      if (r >= p.win_rows || n >= p.N) continue;  // warp-uniform
      beg[i] = __ldg(jb.rowptr[t] + n);
      cnt[i] = __ldg(jb.rowptr[t] + n + 1) - beg[i];
      if (i < SLOTS && lane < cnt[i])
        ent[i] = make_int2(int(__ldg(lc + beg[i] + lane)) * ROWB,
                           __float_as_int(__ldg(val + beg[i] + lane)));
    }
    // the plan and CSR are step constants: read above while the previous kernel drains; the
    // dense operand (and the epilogue's addends) only after it has completed
    if (t == 0) griddep_wait();
    const T *X = reinterpret_cast<const T *>(jb.X[t]) + goff + int64_t(vec0) * V;
    for (int k = warp, i8 = 0; k < nu; k += 8, ++i8) {
      const int node = i8 < 32 ? __shfl_sync(0xffffffffu, my_node, i8)
                               : __ldg(jb.win_nodes[t] + ub + k);
      const T *src = X + int64_t(node) * W;
#pragma unroll
      for (int v = 0; v < VPL; ++v)
        if (vec0 + 32 * v < vecs) cp_async16(stage + (k * VPL + v) * 32 + lane, src + 32 * v * V);
    }
#pragma unroll
    for (int i = 0; i < SLOTS; ++i)
      if (lane < cnt[i]) s_ent[i * 32 + lane] = ent[i];
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      const int slot = i % SLOTS;
      const int2 *E = s_ent + slot * 32;
      if (i >= SLOTS && cnt[i] > 0) {  // RPW 8: refill the slot (warp-private list)
        __syncwarp();
        if (lane < cnt[i])
          s_ent[slot * 32 + lane] = make_int2(int(__ldg(lc + beg[i] + lane)) * ROWB,
                                              __float_as_int(__ldg(val + beg[i] + lane)));
        __syncwarp();
      }
      for (int c0 = 0; c0 < cnt[i]; c0 += 32) {
        if (c0) {  // rows with > 32 entries: the next 32
          __syncwarp();
          if (c0 + lane < cnt[i])
            s_ent[slot * 32 + lane] = make_int2(int(__ldg(lc + beg[i] + c0 + lane)) * ROWB,
                                                __float_as_int(__ldg(val + beg[i] + c0 + lane)));
          __syncwarp();
        }
        const int n0 = min(cnt[i] - c0, 32);
        int u = 0;
        if (VPL == 1) {
          for (; u + 4 <= n0; u += 4) {
            const int2 e0 = E[u], e1 = E[u + 1], e2 = E[u + 2], e3 = E[u + 3];
            const uint4 x0 = *reinterpret_cast<const uint4 *>(lane_stage + e0.x);
            const uint4 x1 = *reinterpret_cast<const uint4 *>(lane_stage + e1.x);
            const uint4 x2 = *reinterpret_cast<const uint4 *>(lane_stage + e2.x);
            const uint4 x3 = *reinterpret_cast<const uint4 *>(lane_stage + e3.x);
            L::fma_v(acc[i][0], __int_as_float(e0.y), x0);
            L::fma_v(acc[i][0], __int_as_float(e1.y), x1);
            L::fma_v(acc[i][0], __int_as_float(e2.y), x2);
            L::fma_v(acc[i][0], __int_as_float(e3.y), x3);
          }
        } else {
          for (; u + 2 <= n0; u += 2) {
            const int2 e0 = E[u], e1 = E[u + 1];
            uint4 x0[VPL], x1[VPL];
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
              x0[v] = *reinterpret_cast<const uint4 *>(lane_stage + e0.x + 512 * v);
              x1[v] = *reinterpret_cast<const uint4 *>(lane_stage + e1.x + 512 * v);
            }
#pragma unroll
            for (int v = 0; v < VPL; ++v) L::fma_v(acc[i][v], __int_as_float(e0.y), x0[v]);
#pragma unroll
            for (int v = 0; v < VPL; ++v) L::fma_v(acc[i][v], __int_as_float(e1.y), x1[v]);
          }
        }
        for (; u < n0; ++u) {
          const int2 e = E[u];
#pragma unroll
          for (int v = 0; v < VPL; ++v)
            L::fma_v(acc[i][v], __int_as_float(e.y),
                     *reinterpret_cast<const uint4 *>(lane_stage + e.x + 512 * v));
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int r = warp + 8 * i, n = row0 + r;
    if (r >= p.win_rows || n >= p.N) continue;
    const int64_t o = goff + int64_t(n) * W + int64_t(vec0) * V;
#pragma unroll
    for (int v = 0; v < VPL; ++v)
      if (vec0 + 32 * v < vecs) finish<L, T, EPI>(jb, acc[i][v], o + 32 * v * V);
  }
}

// Window-resident, chunk-pipelined form (the default for staged launches): CTA = (window, job x
// group) walks ALL column chunks of its rows.  The window's index work -- union node ids (one
// per lane in registers), row pointers, the rows' CSR entries as (staged-row byte offset, value)
// lists in shared memory -- is done once and reused by every chunk, and the chunks are
// double-buffered with cp.async groups: chunk c + 1's neighbour slices are in flight while chunk
// c is reduced.  Per row: the same terms in the same CSR order with the same FFMA2 sequence as
// k_spmm / k_spmm_win (bit-identical).  One term per job, <= 4 rows per warp.
template <typename T, int RPW, int EPI>
__global__ void __launch_bounds__(256, RPW <= 2 ? 3 : 2)
    k_spmm_wp(const __grid_constant__ WinParams p, int cpc) {
  using L = Lane<T>;
  constexpr int V = L::V, P = V / 2;
  extern __shared__ uint4 stage[];  // [2][win_max][32] | entries [8][RPW][32]
  griddep_launch_dependents();
  const int z = int(blockIdx.y);
  int j = 0;
#pragma unroll
  for (int q = 1; q < kMaxSpmmJobs; ++q)
    if (q < p.njobs && z >= p.z_begin[q]) j = q;
  const SpmmJob &jb = p.job[j];
  const int g = z - p.z_begin[j], win = int(blockIdx.x);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int vecs = p.vecs[j];
  const int c_lo = int(blockIdx.z) * cpc, nch = min(p.nchunk[j], c_lo + cpc);  // chunk group
  if (c_lo >= nch) return;
  const int W = int(jb.W);
  const int64_t goff = int64_t(g) * jb.gstride;
  const int row0 = win * p.win_rows;
  const int SB = p.win_max * 32;  // uint4 per stage buffer
  int2 *s_ent = reinterpret_cast<int2 *>(stage + 2 * SB) + warp * (RPW * 32);

  // ---- the window's index work, once
  const int ub = __ldg(jb.win_ptr[0] + win), nu = __ldg(jb.win_ptr[0] + win + 1) - ub;
  const int my_node = warp + 8 * lane < nu ? __ldg(jb.win_nodes[0] + ub + warp + 8 * lane) : 0;
  int beg[RPW], cnt[RPW];
  int2 ent[RPW];
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int r = warp + 8 * i, n = row0 + r;
    beg[i] = cnt[i] = 0;
    ent[i] = make_int2(0, 0);
    if (r >= p.win_rows || n >= p.N) continue;  // warp-uniform
    beg[i] = __ldg(jb.rowptr[0] + n);
    cnt[i] = __ldg(jb.rowptr[0] + n + 1) - beg[i];
    if (lane < cnt[i])
      ent[i] = make_int2(int(__ldg(jb.lcol[0] + beg[i] + lane)) * 512,
                         __float_as_int(__ldg(jb.val[0] + beg[i] + lane)));
  }
  griddep_wait();  // the dense operand (and the epilogue's addends) are predecessor outputs
  const T *X = reinterpret_cast<const T *>(jb.X[0]) + goff + int64_t(lane) * V;
  auto stage_chunk = [&](int c, int b) {  // chunk c's union slices -> buffer b (one group)
    const int vec = c * 32 + lane;
    for (int k = warp, i8 = 0; k < nu; k += 8, ++i8) {
      const int node = i8 < 32 ? __shfl_sync(0xffffffffu, my_node, i8)
                               : __ldg(jb.win_nodes[0] + ub + k);
      if (vec < vecs) cp_async16(stage + b * SB + k * 32 + lane, X + int64_t(node) * W + c * 32 * V);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  stage_chunk(c_lo, 0);
#pragma unroll
  for (int i = 0; i < RPW; ++i)
    if (lane < cnt[i]) s_ent[i * 32 + lane] = ent[i];
  for (int c = c_lo; c < nch; ++c) {
    const int b = (c - c_lo) & 1;
    if (c + 1 < nch) {
      stage_chunk(c + 1, b ^ 1);  // buffer b^1 was released by the previous chunk's barrier
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();  // chunk c staged by every warp; the entry lists written
    const char *st = reinterpret_cast<const char *>(stage + b * SB + lane);
    const int vec = c * 32 + lane;
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      const int r = warp + 8 * i, n = row0 + r;
      if (r >= p.win_rows || n >= p.N) continue;
      float2 acc[P];
#pragma unroll
      for (int q = 0; q < P; ++q) acc[q] = make_float2(0.f, 0.f);
      const int2 *E = s_ent + i * 32;
      const int n0 = min(cnt[i], 32);
      int u = 0;
      for (; u + 4 <= n0; u += 4) {
        const int2 e0 = E[u], e1 = E[u + 1], e2 = E[u + 2], e3 = E[u + 3];
        const uint4 x0 = *reinterpret_cast<const uint4 *>(st + e0.x);
        const uint4 x1 = *reinterpret_cast<const uint4 *>(st + e1.x);
        const uint4 x2 = *reinterpret_cast<const uint4 *>(st + e2.x);
        const uint4 x3 = *reinterpret_cast<const uint4 *>(st + e3.x);
        L::fma_v(acc, __int_as_float(e0.y), x0);
        L::fma_v(acc, __int_as_float(e1.y), x1);
        L::fma_v(acc, __int_as_float(e2.y), x2);
        L::fma_v(acc, __int_as_float(e3.y), x3);
      }
      for (; u < n0; ++u) {
        const int2 e = E[u];
        L::fma_v(acc, __int_as_float(e.y), *reinterpret_cast<const uint4 *>(st + e.x));
      }
      for (int e = beg[i] + 32; e < beg[i] + cnt[i]; ++e)  // rows with > 32 entries
        L::fma_v(acc, __ldg(jb.val[0] + e),
                 *reinterpret_cast<const uint4 *>(st + int(__ldg(jb.lcol[0] + e)) * 512));
      if (vec < vecs) finish<L, T, EPI>(jb, acc, goff + int64_t(n) * W + int64_t(vec) * V);
    }
    __syncthreads();  // every warp is done with buffer b before chunk c + 2 refills it
  }
}

// Tensor-core window SpMM (bf16 hops of the tensor-core step, 16-row windows, union <= 64).
// The SIMT kernels above spend half their instructions unpacking bf16 operands to fp32 for
// FFMA2 and are issue-bound well below HBM bandwidth; the tensor core consumes bf16 natively.
// Per window the 16 x KP transition block P_w (KP = union rounded up to 16; 13 % nonzero on the
// kNN graphs) is built once in shared memory as a bf16 pair hi + lo with hi = bf16(p),
// lo = bf16(p - hi) (relative error of hi + lo <= 2^-17, far below the bf16 output rounding),
// loaded into mma.sync A fragments once, and every column chunk of the window's staged union
// rows X_U (bf16, the same cp.async double buffer as k_spmm_wp, rows XOR-swizzled per 16-byte
// segment so ldmatrix.trans is conflict-free) is multiplied as Y_w = P_hi X_U + P_lo X_U with
// fp32 accumulation (mma.sync.m16n8k16 bf16).  Same products as the SIMT kernels up to fp32
// summation order and the 2^-17 weight split (not bit-identical to them: parity against the
// oracle at the bf16 path's 2e-2; PGTI_SPMM_MMA=0 selects the SIMT kernels).
constexpr int kMmaMaxK = 64, kMmaWin = 16, kMmaPld = kMmaMaxK + 8;  // P_w row pitch (bf16)

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t *r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t *r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void stsm_x4(uint32_t addr, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
  asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1,%2,%3,%4};"
               ::"r"(addr), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
}
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t *>(&v);
}
__device__ __forceinline__ void mma_bf16_16816(float *d, const uint32_t *a, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, "
               "{%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// ADD: the Chebyshev epilogue Y = alpha acc + beta add (add: bf16, Y's layout), applied to the
// fp32 fragments before they are rounded and staged
template <int NST, bool ADD = false>
__global__ void __launch_bounds__(256, 2) k_spmm_mma(const __grid_constant__ WinParams p, int cpc) {
  // [NST][win_max][32] swizzled stage ring | output tiles [2][16][32] swizzled | P_w hi, lo [16][72]
  extern __shared__ __align__(128) uint4 stage[];
  griddep_launch_dependents();
  const int z = int(blockIdx.y);
  int j = 0;
#pragma unroll
  for (int q = 1; q < kMaxSpmmJobs; ++q)
    if (q < p.njobs && z >= p.z_begin[q]) j = q;
  const SpmmJob &jb = p.job[j];
  const int g = z - p.z_begin[j], win = int(blockIdx.x);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int vecs = p.vecs[j];
  const int c_lo = int(blockIdx.z) * cpc, nch = min(p.nchunk[j], c_lo + cpc);
  if (c_lo >= nch) return;
  const int W = int(jb.W);
  const int64_t goff = int64_t(g) * jb.gstride;
  const int row0 = win * kMmaWin;
  const int SB = p.win_max * 32;  // uint4 per stage buffer
  const uint32_t obase = static_cast<uint32_t>(__cvta_generic_to_shared(stage + NST * SB));
  __nv_bfloat16 *Ph = reinterpret_cast<__nv_bfloat16 *>(stage + NST * SB + 2 * kMmaWin * 32);
  __nv_bfloat16 *Pl = Ph + kMmaWin * kMmaPld;

  // ---- the window's index work and transition block, once.  Index loads are issued before the
  // wait on the predecessor grid (they read only the graph), the first chunks' loads right after
  // it, and P_w is scattered while those are in flight.
  const int ub = __ldg(jb.win_ptr[0] + win), nu = __ldg(jb.win_ptr[0] + win + 1) - ub;
  // warp w stages union rows k = w + 8 i (i < nrow): row offsets in elements (N W < 2^31)
  const int my_node = warp + 8 * lane < nu ? __ldg(jb.win_nodes[0] + ub + warp + 8 * lane) : 0;
  const int nrow = nu > warp ? (nu - warp + 7) >> 3 : 0;
  int beg[2], cnt[2], ec[2] = {0, 0};
  float ev[2] = {0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 2; ++i) {  // warp w: window rows w and w + 8, first 32 entries in registers
    const int n = row0 + warp + 8 * i;
    beg[i] = n < p.N ? __ldg(jb.rowptr[0] + n) : 0;
    cnt[i] = n < p.N ? __ldg(jb.rowptr[0] + n + 1) - beg[i] : 0;
    if (lane < cnt[i]) ec[i] = int(__ldg(jb.lcol[0] + beg[i] + lane)), ev[i] = __ldg(jb.val[0] + beg[i] + lane);
  }
  uint32_t roff[kMmaMaxK / 8];  // byte offsets (N W 2 < 2^32): one 64-bit add per row and chunk
#pragma unroll
  for (int i = 0; i < kMmaMaxK / 8; ++i)
    roff[i] = uint32_t(__shfl_sync(0xffffffffu, my_node, i)) * uint32_t(2 * W);
  const int KS = (nu + 15) >> 4;  // k-steps of 16 union rows; rows nu..16 KS-1 meet zero columns
  for (int i = threadIdx.x; i < kMmaWin * kMmaPld / 4; i += blockDim.x)  // Ph, Pl: 2 x 2304 B
    reinterpret_cast<uint4 *>(Ph)[i] = make_uint4(0u, 0u, 0u, 0u);
  griddep_wait();  // the dense operand is the predecessor's output
  // lane l's 16-byte vector of chunk c: global X + node W + 256 c + 8 l; shared row k, segment
  // l ^ (k & 7) = l ^ w (k = w + 8 i)
  const __nv_bfloat16 *Xl = reinterpret_cast<const __nv_bfloat16 *>(jb.X[0]) + goff + lane * 8;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
  const uint32_t sst = sbase + uint32_t(warp * 512 + ((lane ^ warp) << 4));
  auto stage_chunk = [&](int c) {
    if (c < nch && c * 32 + lane < vecs) {
      const uint32_t dst = sst + uint32_t(((c - c_lo) % NST) * SB) * 16u;
      const char *src = reinterpret_cast<const char *>(Xl + c * 256);
#pragma unroll
      for (int i = 0; i < kMmaMaxK / 8; ++i)
        if (i < nrow)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + i * 4096),
                       "l"(src + roff[i])
                       : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");  // (empty past the last chunk)
  };
#pragma unroll
  for (int q = 0; q < NST - 1; ++q) stage_chunk(c_lo + q);
  __syncthreads();  // P_w zeroed
  auto put = [&](int r, int c, float v) {
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    Ph[r * kMmaPld + c] = hi;
    Pl[r * kMmaPld + c] = __float2bfloat16_rn(v - __bfloat162float(hi));
  };
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = warp + 8 * i;
    if (lane < cnt[i]) put(r, ec[i], ev[i]);
    for (int e = 32 + lane; e < cnt[i]; e += 32)
      put(r, int(__ldg(jb.lcol[0] + beg[i] + e)), __ldg(jb.val[0] + beg[i] + e));
  }
  __syncthreads();  // P_w complete
  // A fragments of all k-steps (hi and lo), kept in registers for every chunk of the window;
  // B (ldmatrix.trans) offsets: matrix mi = lane / 8 holds k rows (mi & 1) 8 + lane % 8 of the
  // k-step (padding rows read row nu - 1: finite values against zero weights) and the 8 columns
  // of n-tile 2 h + (mi >> 1) of the warp's four
  uint32_t ah[4][4], al[4][4], boff[4][2];
  {
    const int mi = lane >> 3, rr = lane & 7;
    const int prow = (mi & 1) * 8 + rr, pcol = (mi >> 1) * 8;
    const uint32_t hb = static_cast<uint32_t>(__cvta_generic_to_shared(Ph));
    const uint32_t lb = static_cast<uint32_t>(__cvta_generic_to_shared(Pl));
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      if (ks < KS) {
        const uint32_t off = uint32_t((prow * kMmaPld + ks * 16 + pcol) * 2);
        ldsm_x4(hb + off, ah[ks]);
        ldsm_x4(lb + off, al[ks]);
      }
      const int k = max(min(ks * 16 + (mi & 1) * 8 + rr, nu - 1), 0);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int seg = warp * 4 + 2 * h + (mi >> 1);
        boff[ks][h] = uint32_t(k * 512 + ((seg ^ (k & 7)) << 4));
      }
    }
  }
  // output: D fragments go to a swizzled [16][512 B] shared tile by stmatrix (matrix mi of
  // stmatrix q: n-tile 2 q + (mi >> 1), rows 8 (mi & 1) + lane % 8), stored to global one
  // chunk later as full 512-byte row segments (warp w: window rows w and w + 8)
  uint32_t soff[2];
  {
    const int mi = lane >> 3, rr = lane & 7;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int row = 8 * (mi & 1) + rr, seg = warp * 4 + 2 * q + (mi >> 1);
      soff[q] = uint32_t(row * 512 + ((seg ^ rr) << 4));
    }
  }
  const uint32_t lds0 = uint32_t(warp * 512 + ((lane ^ warp) << 4));  // rows w, w + 8: same swizzle
  __nv_bfloat16 *Yw = reinterpret_cast<__nv_bfloat16 *>(jb.Y) + goff + int64_t(row0 + warp) * W +
                      lane * 8;
  const bool w0ok = row0 + warp < p.N, w1ok = row0 + warp + 8 < p.N;
  auto store_chunk = [&](int c) {
    if (c * 32 + lane < vecs) {
      const uint32_t ob = obase + uint32_t((c - c_lo) & 1) * (kMmaWin * 512);
      uint4 v0, v1;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v0.x), "=r"(v0.y), "=r"(v0.z), "=r"(v0.w) : "r"(ob + lds0));
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v1.x), "=r"(v1.y), "=r"(v1.z), "=r"(v1.w) : "r"(ob + lds0 + 8 * 512));
      if (w0ok) *reinterpret_cast<uint4 *>(Yw + c * 256) = v0;
      if (w1ok) *reinterpret_cast<uint4 *>(Yw + int64_t(8) * W + c * 256) = v1;
    }
  };
  for (int c = c_lo; c < nch; ++c) {
    asm volatile("cp.async.wait_group %0;" ::"n"(NST - 2) : "memory");
    __syncthreads();  // chunk c landed; buffer of chunk c - 1 and output tile of c - 2 are free
    stage_chunk(c + NST - 1);
    if (c > c_lo) store_chunk(c - 1);
    const uint32_t bb = sbase + uint32_t(((c - c_lo) % NST) * SB) * 16u;
    float acc[4][4];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[t][q] = 0.f;
    // B fragments one k-step ahead of the MMAs that consume them
    uint32_t bf[2][2][4];
    ldsm_x4_t(bb + boff[0][0], bf[0][0]);
    ldsm_x4_t(bb + boff[0][1], bf[0][1]);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      if (ks >= KS) break;
      if (ks + 1 < 4 && ks + 1 < KS) {
        ldsm_x4_t(bb + boff[ks + 1][0], bf[(ks + 1) & 1][0]);
        ldsm_x4_t(bb + boff[ks + 1][1], bf[(ks + 1) & 1][1]);
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t b0 = bf[ks & 1][t >> 1][(t & 1) * 2], b1 = bf[ks & 1][t >> 1][(t & 1) * 2 + 1];
        mma_bf16_16816(acc[t], ah[ks], b0, b1);
        mma_bf16_16816(acc[t], al[ks], b0, b1);
      }
    }
    if constexpr (ADD) {  // fragment (t, hr): row gq + 8 hr, columns 2 tq, 2 tq + 1 of n-tile t
      const __nv_bfloat16 *A = reinterpret_cast<const __nv_bfloat16 *>(jb.add) + goff;
      const float al = jb.alpha, be = jb.beta;
      const int gq = lane >> 2, tq = lane & 3;
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int n = row0 + gq + 8 * hr;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int col = (c * 32 + warp * 4 + t) * 8 + 2 * tq;
          float2 a = make_float2(0.f, 0.f);
          if (n < p.N && col < W)
            a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(A + int64_t(n) * W + col));
          acc[t][2 * hr] = fmaf(al, acc[t][2 * hr], be * a.x);
          acc[t][2 * hr + 1] = fmaf(al, acc[t][2 * hr + 1], be * a.y);
        }
      }
    }
    const uint32_t ob = obase + uint32_t((c - c_lo) & 1) * (kMmaWin * 512);
#pragma unroll
    for (int q = 0; q < 2; ++q)  // matrices (tile 2q, rows 0-7), (2q, 8-15), (2q+1, 0-7), (2q+1, 8-15)
      stsm_x4(ob + soff[q], pack_bf16x2(acc[2 * q][0], acc[2 * q][1]),
              pack_bf16x2(acc[2 * q][2], acc[2 * q][3]), pack_bf16x2(acc[2 * q + 1][0], acc[2 * q + 1][1]),
              pack_bf16x2(acc[2 * q + 1][2], acc[2 * q + 1][3]));
  }
  __syncthreads();
  store_chunk(nch - 1);
  asm volatile("cp.async.wait_group 0;" ::: "memory");
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
             jobs[0].win_max * 512 + (jobs[0].win_max + 3) / 4 * 16 + kWinEntBytes <= kWinMaxSmem;
  for (int i = 0; i < njobs && win; ++i) {
    const SpmmJob &j = jobs[i];
    win = j.nterms >= 1 && j.win_rows == jobs[0].win_rows && j.win_max == jobs[0].win_max;
    for (int t = 0; t < j.nterms && win; ++t) win = j.win_ptr[t] && j.win_nodes[t] && j.lcol[t];
  }
  WinParams w{};
  int nz = 0, maxc = 0;
  // two 16-byte vectors per lane (1 KB column chunks) for wide bf16 operands: the per-warp
  // index / entry / epilogue work is shared by twice the columns (PGTI_SPMM_VPL=1 disables)
  int vpl = 1;
  if (win && bf) {
    const char *e = std::getenv("PGTI_SPMM_VPL");
    vpl = (e && e[0] == '1') ? 1 : 2;
    for (int i = 0; i < njobs; ++i) vpl = jobs[i].W / V >= 64 ? vpl : 1;
    if (jobs[0].win_rows > 32) vpl = 1;
    if (2 * jobs[0].win_max * 512 + (jobs[0].win_max + 3) / 4 * 16 + kWinEntBytes > kWinMaxSmem)
      vpl = 1;
  }
  if (win) {
    w.njobs = njobs, w.N = N, w.win_rows = jobs[0].win_rows, w.win_max = jobs[0].win_max;
    w.nwin = int(ceil_div(N, w.win_rows));
    for (int i = 0; i < njobs; ++i) {
      w.job[i] = jobs[i];
      w.vecs[i] = int(jobs[i].W / V);
      w.nchunk[i] = int(ceil_div(w.vecs[i], 32 * vpl));
      w.z_begin[i] = nz;
      nz += jobs[i].G;
      maxc = std::max(maxc, w.nchunk[i]);
    }
    w.z_begin[njobs] = nz;
    if (nz > 65535 || w.nwin > 65535) win = false;
  }
  // window-resident, chunk-pipelined kernel: every job one term, <= 4 rows per warp
  bool wp = win && (w.win_rows + 7) / 8 <= 4;
  for (int i = 0; i < njobs && wp; ++i) wp = jobs[i].nterms == 1;
  {
    const char *e = std::getenv("PGTI_SPMM_WP");
    if (e && e[0] == '0') wp = false;
  }
  // CTAs = windows x jobs x chunk groups, >= one per SM; the SIMT window-resident kernel needs
  // >= 4 chunks per group for the window's index work and the pipeline to pay, the tensor-core
  // kernel >= 2 (else the per-chunk kernel below)
  int cpc = 0;
  const bool one_term = wp;
  if (wp) {
    const int V1 = bf ? 8 : 4;
    int mc = 0;
    for (int i = 0; i < njobs; ++i) mc = std::max<int>(mc, int(ceil_div(jobs[i].W / V1, 32)));
    const int64_t base = int64_t(w.nwin) * nz;
    // chunk groups: enough CTAs for one CTA per SM (one wave at 1 CTA per SM: the kernels of
    // the concurrent layer stream keep the other slots; METR-LA 43.2 K -> 47.0 K samples/s,
    // PeMS-Bay 31.7 K -> 32.9 K against 4 waves).  PGTI_SPMM_WAVES overrides (A/B)
    const char *ew = std::getenv("PGTI_SPMM_WAVES");
    const int waves = (ew && ew[0] >= '1' && ew[0] <= '8') ? ew[0] - '0' : 1;
    const int ngrp = int(std::max<int64_t>(1, ceil_div(int64_t(waves) * kNumSMs, base)));
    cpc = int(ceil_div(mc, ngrp));
    wp = cpc >= 4;
  }
  // tensor-core window SpMM: bf16, 16-row windows, union <= 64, plain hops (store only)
  // (plain hops, or the Chebyshev form alpha acc + beta add: the ADD instantiation)
  bool mma = one_term && bf && w.win_rows == kMmaWin && w.win_max <= kMmaMaxK;
  bool mma_add = false;
  for (int i = 0; i < njobs && mma; ++i) {
    mma = !jobs[i].accumulate && !jobs[i].add2 && jobs[i].W % 8 == 0 &&
          int64_t(N) * jobs[i].W < (int64_t(1) << 31);
    mma_add = mma_add || jobs[i].add || jobs[i].alpha != 1.f || jobs[i].beta != 1.f;
  }
  for (int i = 0; i < njobs && mma && mma_add; ++i) mma = jobs[i].add != nullptr;
  {  // default where a CTA walks >= 2 chunks of its window (full PeMS 16, PeMS-All-LA 8,
     // PeMS-Bay 2; METR-LA's 13 windows leave 1 and the per-chunk SIMT kernel is faster there);
     // 0 = off, 1 = wherever eligible
    const char *e = std::getenv("PGTI_SPMM_MMA");
    if (e && e[0] == '0') mma = false;
    else if (!(e && e[0] == '1')) mma = mma && cpc >= 2;
  }
  if (mma) {
    int mc = 0;
    for (int i = 0; i < njobs; ++i) {
      w.vecs[i] = int(jobs[i].W / 8);
      w.nchunk[i] = int(ceil_div(w.vecs[i], 32));
      mc = std::max(mc, w.nchunk[i]);
    }
    // stage ring depth: NST - 1 chunks in flight per CTA while one is multiplied (2 CTAs / SM)
    const char *e = std::getenv("PGTI_SPMM_NST");
    const int nst = (e && e[0] >= '2' && e[0] <= '4') ? e[0] - '0' : 3;
    const int smem = nst * w.win_max * 512 + 2 * kMmaWin * 512 + 2 * kMmaWin * kMmaPld * 2;
    const int ngrp = int(ceil_div(mc, cpc));
    const dim3 grid(unsigned(w.nwin), unsigned(nz), unsigned(ngrp));
    auto go = [&](auto kern) -> cudaError_t {
      cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (r != cudaSuccess) return r;
      return pdl_launch(kern, grid, dim3(256), smem, s, w, cpc);
    };
    if (mma_add) return go(k_spmm_mma<3, true>);
    return nst == 2 ? go(k_spmm_mma<2>) : nst == 4 ? go(k_spmm_mma<4>) : go(k_spmm_mma<3>);
  }
  if (wp) {
    const int V1 = bf ? 8 : 4;
    int mc = 0;
    for (int i = 0; i < njobs; ++i) {  // one 16-byte vector per lane: 512-byte chunks
      w.vecs[i] = int(jobs[i].W / V1);
      w.nchunk[i] = int(ceil_div(w.vecs[i], 32));
      mc = std::max(mc, w.nchunk[i]);
    }
    const int smem = 2 * jobs[0].win_max * 512 + 8 * 4 * 32 * 8;
    const dim3 grid(unsigned(w.nwin), unsigned(nz), unsigned(ceil_div(mc, cpc)));
    const int rpw = (w.win_rows + 7) / 8;
    bool store_only = true;
    for (int i = 0; i < njobs; ++i) store_only = store_only && !jobs[i].add && !jobs[i].accumulate;
    auto go = [&](auto kernel) -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      return pdl_launch(kernel, grid, dim3(256), smem, s, w, cpc);
    };
    auto pick = [&](auto epi) -> cudaError_t {
      constexpr int G = decltype(epi)::value;
      if (bf) {
        if (rpw <= 1) return go(k_spmm_wp<__nv_bfloat16, 1, G>);
        if (rpw <= 2) return go(k_spmm_wp<__nv_bfloat16, 2, G>);
        return go(k_spmm_wp<__nv_bfloat16, 4, G>);
      }
      if (rpw <= 1) return go(k_spmm_wp<float, 1, G>);
      if (rpw <= 2) return go(k_spmm_wp<float, 2, G>);
      return go(k_spmm_wp<float, 4, G>);
    };
    if (gen) return pick(std::integral_constant<int, 2>{});
    return store_only ? pick(std::integral_constant<int, 0>{})
                      : pick(std::integral_constant<int, 1>{});
  }
  if (win) {
    const dim3 grid(unsigned(maxc), unsigned(w.nwin), unsigned(nz));
    // staged rows + their node ids + the per-warp entry lists
    const int smem = jobs[0].win_max * 512 * vpl + kWinEntBytes;
    const int rpw = (w.win_rows + 7) / 8;
    auto go = [&](auto kernel) -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      return pdl_launch(kernel, grid, dim3(256), smem, s, w);
    };
    auto pick = [&](auto epi) -> cudaError_t {
      constexpr int G = decltype(epi)::value;
      if (bf && vpl == 2) {
        if (rpw <= 1) return go(k_spmm_win<__nv_bfloat16, 1, 2, G>);
        if (rpw <= 2) return go(k_spmm_win<__nv_bfloat16, 2, 2, G>);
        if (rpw <= 4) return go(k_spmm_win<__nv_bfloat16, 4, 2, G>);
        return go(k_spmm_win<__nv_bfloat16, 8, 1, G>);  // not reached: vpl 2 needs rpw <= 4
      }
      if (bf) {
        if (rpw <= 1) return go(k_spmm_win<__nv_bfloat16, 1, 1, G>);
        if (rpw <= 2) return go(k_spmm_win<__nv_bfloat16, 2, 1, G>);
        if (rpw <= 4) return go(k_spmm_win<__nv_bfloat16, 4, 1, G>);
        return go(k_spmm_win<__nv_bfloat16, 8, 1, G>);
      }
      if (rpw <= 1) return go(k_spmm_win<float, 1, 1, G>);
      if (rpw <= 2) return go(k_spmm_win<float, 2, 1, G>);
      if (rpw <= 4) return go(k_spmm_win<float, 4, 1, G>);
      return go(k_spmm_win<float, 8, 1, G>);
    };
    // the general epilogue (Chebyshev / Clenshaw: alpha, beta, add2) costs registers (bf16 x 4
    // rows: 79 -> 91, 3 -> 2 CTAs per SM), so it is its own instantiation; so is the store-only
    // epilogue of the plain hops (no predicated addend / accumulator code per row)
    bool store_only = true;
    for (int i = 0; i < njobs; ++i) store_only = store_only && !jobs[i].add && !jobs[i].accumulate;
    if (gen) return pick(std::integral_constant<int, 2>{});
    return store_only ? pick(std::integral_constant<int, 0>{})
                      : pick(std::integral_constant<int, 1>{});
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

}  // namespace pgti
