// Skinny weight gradients (bias rows, layer-0 input rows, readout W_out / b_out):
// out[s][j] = sum_t sum_r S_t[r][s] G_t[r][j] with ns <= 12 small rows and a wide G.
// Memory-bound on G (read once, coalesced along j); the small operand is staged per 64-row tile
// in shared memory and broadcast.  Row chunks never cross a time step; chunk partials are summed
// in a fixed order (bitwise reproducible).
#include <type_traits>

#include "kernels.cuh"
#include "profile.cuh"
#include "tc_ptx.cuh"

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

// Thread = VEC consecutive columns of a G row, tpr = NG / VEC threads per row, 256 / tpr row
// groups per CTA.  G is streamed in 128-row tiles (one contiguous 16-32 KB block: G rows are
// [R][NG]) by a TMA bulk copy into a double-buffered shared tile, the next tile in flight while
// the current one is reduced -- the load is one instruction and the bytes in flight do not
// depend on registers.  The small operand's next tile is loaded into registers at the same time
// and stored after the reduction (the per-thread element -> (row, column, offset) map is
// computed once).  Per row a thread reads its VEC columns and the row's ns small values (LDS.128
// broadcast) and accumulates ns x VEC products with FFMA2 (the bias row of kSmallBiasX is S =
// 1).  Row groups are folded in a fixed order in shared memory, chunk partials by
// k_small_reduce in a fixed order (reproducible).
constexpr int kST = 128;                                  // rows per staged tile
constexpr int kSE = (kST * kSmallMax + kThr - 1) / kThr;  // staged small elements per thread
constexpr int kGTile = kST * 128 * 2;                     // G tile bytes (128 bf16 / 64 fp32)

template <typename T, int NS, int VEC>
__global__ void __launch_bounds__(kThr, 2) k_small_wgrad(const __grid_constant__ SmallWgrad p, Plan q) {
  extern __shared__ __align__(128) uint8_t gsm[];  // [2][kGTile] G tiles
  __shared__ __align__(16) float S[2][kST][kSmallMax];
  __shared__ __align__(16) float red[kSmallMax * 128];
  __shared__ __align__(8) uint64_t mbar[2];
  griddep_launch_dependents();
  const int chunk = blockIdx.x, t = chunk / q.cpt;
  const int r0 = (chunk - t * q.cpt) * q.RC, r1 = min(p.R, r0 + q.RC);
  const int tpr = p.NG / VEC, rgs = kThr / tpr;
  const int cg = threadIdx.x % tpr, rg = threadIdx.x / tpr;
  const bool readout = p.mode == kSmallReadout;
  // this thread's staged small elements: tile row << 8 | column, source offset (-1: constant 1)
  int e_rs[kSE], e_off[kSE];
  const float *src = readout ? p.dy + int64_t(t) * p.R * p.F_out : p.Dx + t * p.dx_tstride;
  const int rstride = readout ? p.F_out : p.F;
#pragma unroll
  for (int k = 0; k < kSE; ++k) {
    const int e = threadIdx.x + k * kThr, rr = e / q.ns, sl = e - rr * q.ns;
    e_rs[k] = rr << 8 | sl;
    if (readout) {
      e_off[k] = sl;
    } else if (sl == q.ns - 1) {
      e_off[k] = -1;
    } else {
      const int m = sl / p.F, f = sl - m * p.F;
      e_off[k] = int(m * p.dx_mstride) + f;
    }
  }
  float2 acc[NS][VEC / 2];
  float accb[NS];  // readout: the ones column (b_out = sum dy), kept by the cg == 0 threads
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    accb[s] = 0.f;
#pragma unroll
    for (int v = 0; v < VEC / 2; ++v) acc[s][v] = make_float2(0.f, 0.f);
  }
  const T *G = reinterpret_cast<const T *>(std::is_same<T, float>::value
                                               ? static_cast<const void *>(p.G)
                                               : static_cast<const void *>(p.Gb)) +
               t * p.g_tstride;
  const int row_bytes = p.NG * int(sizeof(T));
  float st[kSE];
  auto load_small = [&](int rb) {
    const int nr = min(kST, r1 - rb);
#pragma unroll
    for (int k = 0; k < kSE; ++k) {
      st[k] = 0.f;
      if ((e_rs[k] >> 8) < nr)
        st[k] = e_off[k] < 0 ? 1.0f
                             : __ldg(src + int64_t(rb + (e_rs[k] >> 8)) * rstride + e_off[k]);
    }
  };
  auto store_small = [&](int b) {
#pragma unroll
    for (int k = 0; k < kSE; ++k)
      if ((e_rs[k] >> 8) < kST) S[b][e_rs[k] >> 8][e_rs[k] & 255] = st[k];
  };
  auto issue_g = [&](int rb, int b) {  // thread 0: rows [rb, rb + nr) of G -> tile b
    const uint32_t bytes = uint32_t(min(kST, r1 - rb)) * uint32_t(row_bytes);
    const uint32_t mb = tc::smem_u32(&mbar[b]);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(tc::smem_u32(gsm + b * kGTile)), "l"(G + int64_t(rb) * p.NG), "r"(bytes), "r"(mb)
        : "memory");
  };
  if (threadIdx.x == 0) {
    tc::mbar_init(&mbar[0], 1);
    tc::mbar_init(&mbar[1], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();
  if (r0 < r1) {
    if (threadIdx.x == 0) issue_g(r0, 0);
    load_small(r0);
    store_small(0);
  }
  __syncthreads();
  uint32_t phase = 0u;  // bit b: parity of buffer b's next completion
  for (int rb = r0, b = 0; rb < r1; rb += kST, b ^= 1) {
    const int nr = min(kST, r1 - rb);
    const bool more = rb + kST < r1;
    if (more) {  // both operands of the next tile in flight while this one is reduced
      if (threadIdx.x == 0) issue_g(rb + kST, b ^ 1);
      load_small(rb + kST);
    }
    tc::mbar_wait(&mbar[b], (phase >> b) & 1u);
    phase ^= 1u << b;
    const uint8_t *gt = gsm + b * kGTile + cg * VEC * int(sizeof(T));
#pragma unroll 2
    for (int rr = rg; rr < nr; rr += rgs) {
      float2 g[VEC / 2];
      if constexpr (std::is_same<T, float>::value) {
        const float4 f = *reinterpret_cast<const float4 *>(gt + rr * row_bytes);
        g[0] = make_float2(f.x, f.y), g[1] = make_float2(f.z, f.w);
      } else if constexpr (VEC == 8) {
        const uint4 w = *reinterpret_cast<const uint4 *>(gt + rr * row_bytes);
        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int v = 0; v < 4; ++v)
          g[v] = make_float2(__uint_as_float(ww[v] << 16), __uint_as_float(ww[v] & 0xffff0000u));
      } else if constexpr (VEC == 4) {
        const uint2 w = *reinterpret_cast<const uint2 *>(gt + rr * row_bytes);
        g[0] = make_float2(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u));
        g[1] = make_float2(__uint_as_float(w.y << 16), __uint_as_float(w.y & 0xffff0000u));
      } else {  // VEC 2
        const uint32_t w = *reinterpret_cast<const uint32_t *>(gt + rr * row_bytes);
        g[0] = make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
      }
      float sv[kSmallMax];
      const float4 *Srow = reinterpret_cast<const float4 *>(S[b][rr]);
#pragma unroll
      for (int c = 0; c < (NS + 3) / 4; ++c) {
        const float4 f4 = Srow[c];
        sv[4 * c] = f4.x, sv[4 * c + 1] = f4.y, sv[4 * c + 2] = f4.z, sv[4 * c + 3] = f4.w;
      }
#pragma unroll
      for (int s = 0; s < NS; ++s)
        if (s < q.ns) {
          const float2 ss = make_float2(sv[s], sv[s]);
#pragma unroll
          for (int v = 0; v < VEC / 2; ++v) acc[s][v] = __ffma2_rn(ss, g[v], acc[s][v]);
          if (readout) accb[s] += sv[s];
        }
    }
    if (more) store_small(b ^ 1);  // buffer b^1 was last read before the previous barrier
    __syncthreads();
  }
  // fold the row groups in order: group 0 writes, groups 1.. add in turn
  for (int gi = 0; gi < rgs; ++gi) {
    if (rg == gi)
#pragma unroll
      for (int s = 0; s < NS; ++s)
        if (s < q.ns)
#pragma unroll
          for (int v = 0; v < VEC / 2; ++v) {
            float2 *o = reinterpret_cast<float2 *>(red + s * 128 + cg * VEC) + v;
            *o = gi == 0 ? acc[s][v] : make_float2(o->x + acc[s][v].x, o->y + acc[s][v].y);
          }
    __syncthreads();
  }
  float *out = p.partial + int64_t(chunk) * q.ns * q.ngt;
  for (int i = threadIdx.x; i < q.ns * p.NG; i += kThr) {
    const int sl = i / p.NG, c = i - sl * p.NG;
    out[sl * q.ngt + c] = red[sl * 128 + c];
  }
  if (readout) {  // the ones column: fold the cg == 0 threads' sums in row-group order
    __shared__ float redb[kThr / 2][kSmallMax];
    if (cg == 0)
#pragma unroll
      for (int s = 0; s < NS; ++s) redb[rg][s] = accb[s];
    __syncthreads();
    if (threadIdx.x < q.ns) {
      float bsum = 0.f;
      for (int gi = 0; gi < rgs; ++gi) bsum += redb[gi][threadIdx.x];
      out[threadIdx.x * q.ngt + p.NG] = bsum;
    }
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
  {  // tpr = NG / VEC threads per row must divide the CTA
    const int vec = p.Gb ? (q.ns <= 1 ? 8 : 2) : 4, tpr = p.NG / vec;
    if (p.NG % vec || tpr > kThr || kThr % tpr) return cudaErrorInvalidValue;
    if (int64_t(p.NG) * (p.Gb ? 2 : 4) > 256 || (int64_t(p.NG) * (p.Gb ? 2 : 4)) % 16)
      return cudaErrorInvalidValue;  // G tile rows: 16-byte multiples, <= 256 bytes
  }
  if (int64_t(q.nchunks) * q.ns * q.ngt > p.partial_cap) return cudaErrorInvalidValue;
  if (p.mode == kSmallBiasX && p.Dx && int64_t(p.M) * p.dx_mstride >= (int64_t(1) << 31))
    return cudaErrorInvalidValue;  // 32-bit staging offsets
  cudaError_t e;
  {
    const double tr = double(p.T) * p.R;
    ProfScope prof(kProfGemmWgrad, s, tr * ((p.Gb ? 2.0 : 4.0) * p.NG + 4.0 * q.ns),
                   2.0 * tr * q.ns * q.ngt);
    const dim3 grid(unsigned(q.nchunks)), block(kThr);
    const int smem = 2 * kGTile;
    auto go = [&](auto kernel) -> cudaError_t {
      cudaError_t e2 = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      return e2 != cudaSuccess ? e2 : pdl_launch(kernel, grid, block, smem, s, p, q);
    };
    // bf16 G: 8 columns per thread for the bias-only rows; 2 when 11 small rows are accumulated
    // per column (registers)
    if (p.Gb)
      e = q.ns <= 1 ? go(k_small_wgrad<__nv_bfloat16, 1, 8>)
                    : go(k_small_wgrad<__nv_bfloat16, kSmallMax, 2>);
    else if (q.ns <= 4)  // fp32 G: the readout (ns = F_out <= 4)
      e = q.ns <= 1 ? go(k_small_wgrad<float, 1, 4>) : go(k_small_wgrad<float, 4, 4>);
    else
      e = cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  ProfScope prof(kProfReduce, s, 4.0 * double(q.nchunks + 1) * q.ns * q.ngt,
                 double(q.nchunks) * q.ns * q.ngt);
  return pdl_launch(k_small_reduce, dim3(unsigned(ceil_div(q.ns * q.ngt, 8))), dim3(256), 0, s,
                    p, q);
}

}  // namespace pgti
