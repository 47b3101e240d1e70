// K3: tcgen05 gate GEMMs (bf16 operands staged by TMA into SWIZZLE_128B shared memory, fp32
// accumulators in TMEM, one elected thread issuing tcgen05.mma) with the GRU math fused into
// the epilogue.
//   k_tc_fwd   : multi-block GEMM (forward gates, and the backward "diffuse-then-GEMM" dgrad)
//                10 warps: warp 0 TMA producer, warp 1 TMEM alloc + MMA issuer, warps 2-9
//                epilogue.  Epilogue = TMEM -> registers -> shared-memory tile (the drained
//                pipeline stages are reused) -> coalesced element-wise math and global I/O
//                (consecutive threads touch consecutive columns of a row).
//   k_tc_wgrad : split-K weight gradient, MN-major A (diffusion blocks) and B (gate gradients)
// mbarrier ring between TMA and MMA (full / empty; 4 stages, 3 for two-sub-tile CTAs so two
// CTAs fit per SM and one's epilogue overlaps the other's main loop), one commit barrier
// MMA -> epilogue.
// Equations: Li et al. Eq. 2-3 [ext], PAPER.md P:168, P:222 (readings c1-c7).
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "kernels.cuh"
#include "profile.cuh"
#include "tc_gemm.cuh"
#include "tc_ptx.cuh"

namespace pgti {
namespace {

using namespace tc;
using bf16 = __nv_bfloat16;

constexpr int kBM = 128, kBK = 64, kStages = 4;

struct Barriers {
  uint64_t full[kStages], empty[kStages], tfull;
  uint32_t tmem;
};

template <int A_BYTES, int B_BYTES, int NST = kStages>
__device__ __forceinline__ Barriers *carve(uint8_t *smem) {
  return reinterpret_cast<Barriers *>(smem + NST * (A_BYTES + B_BYTES));
}

// Offset arithmetic on the shared-memory pointer itself (not an integer round trip), so the
// compiler keeps the shared address space and emits STS/LDS instead of generic ST/LD.
__device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  return p + ((1024u - (a & 1023u)) & 1023u);
}

__device__ __forceinline__ void setup(Barriers *bar, uint32_t ncols) {
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar->full[s], 1), mbar_init(&bar->empty[s], 1);
    mbar_init(&bar->tfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&bar->tmem, ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
}

__device__ __forceinline__ void teardown(Barriers *bar, uint32_t ncols) {
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x / 32 == 1) {
    tc_fence_after();
    tmem_dealloc(bar->tmem, ncols);
  }
}

__device__ __forceinline__ float4 ld4(const float *p) { return *reinterpret_cast<const float4 *>(p); }
__device__ __forceinline__ float4 ld4_bf16(const bf16 *p) {
  const uint2 u = *reinterpret_cast<const uint2 *>(p);
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void st4(float *p, float4 v) { *reinterpret_cast<float4 *>(p) = v; }
__device__ __forceinline__ void st4_bf16(bf16 *p, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t *>(&a);
  u.y = *reinterpret_cast<uint32_t *>(&b);
  *reinterpret_cast<uint2 *>(p) = u;
}

// ================================================================== multi-block GEMM
constexpr int kFwdThreads = 320, kEpiThreads = 256;
constexpr int fwd_stages(int nsub) { return nsub == 2 ? 3 : 4; }
constexpr int kTileLd = 68;  // shared epilogue tile pitch (floats): 16-byte rows, spread banks

// named barrier of one epilogue group (8 warps): id 1 + group
__device__ __forceinline__ void epi_bar(int eg = 0) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + eg), "n"(kEpiThreads) : "memory");
}

// ------------------------------------------------------------------ forward GEMM epilogue
// Epilogue
// threads et = 0..255 (warps 2-9: e = warp - 2, q = warp & 3 = TMEM lane quarter, hh = e >> 2 =
// column half).
// (1) While the tile's MMAs run: pull the epilogue's [128 rows][64 fp32] input tiles into L2,
// and stage the layer-0 x part (the tile's 128 rows of the diffused input, the first sub-tile's
// weight rows).  Returns nx = F M (0 when there is no x part).
template <int NSUB, int MODE>
__device__ __forceinline__ int fwd_epi_prepare(const TcFwd &p, int row0, int ct0, int et,
                                               float *wx_s, float *xs_s) {
  const int H = p.H;
  const int nx = (MODE != kEpiBwd && p.Dx) ? p.F * p.M : 0;
  {  // while the MMAs run: pull the epilogue's [128 rows][64 fp32] input tiles into L2
    const int rl = et >> 1, row = row0 + rl;
    auto pf = [&](const float *base, int64_t pitch) {
      if (base && row < p.R)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(base + row * pitch + (et & 1) * 32));
    };
    if (MODE == kEpiGate && ct0 == 0) pf(p.Hprev, H);
    if (MODE == kEpiCand) pf(p.u_in + ct0 * 64, H), pf(p.Hprev ? p.Hprev + ct0 * 64 : nullptr, H);
    if (MODE == kEpiBwd)
      for (int sub = 0; sub < NSUB; ++sub) {
        const int ct = ct0 + sub;
        if (ct == p.fuse_tile) {
          pf(p.Hprev, 64), pf(p.g_dHprev, 64);
          if (row < p.R && !(et & 1))  // r is bf16: one 128-byte line per row
            asm volatile("prefetch.global.L2 [%0];" ::"l"(p.g_r + int64_t(row) * 64));
        } else if (p.dst_acc[ct]) {
          pf(p.dst[ct], 64);
        }
      }
  }
  // layer-0 x part while the MMAs run: the tile's 128 rows of the diffused input and the
  // first sub-tile's weight rows (visible to every epilogue thread after phase 1's barrier)
  for (int i = et; i < nx * 64; i += kEpiThreads) {
    const int mf = i / 64, j = i % 64, m = mf / p.F, f = mf % p.F;
    wx_s[i] = __ldg(p.Wx + int64_t(m * p.C_in + f) * p.Nout + ct0 * 64 + j);
  }
  for (int i = et; i < nx * kBM; i += kEpiThreads) {
    const int rl = i / nx, mf = i - rl * nx, m = mf / p.F, f = mf - m * p.F;
    xs_s[i] = row0 + rl < p.R ? __ldg(p.Dx + m * p.dx_mstride + int64_t(row0 + rl) * p.F + f) : 0.f;
  }
  return nx;
}

// (2) The tile's epilogue from the TMEM accumulator at tacc: per 64-column sub-tile, TMEM ->
// registers -> the shared tile (phase 1), then the coalesced element-wise math and global I/O
// (phase 2).  `drained` (nullable): arrived on (one thread) once every TMEM load of the tile is
// complete, so the MMA warp may reuse the accumulator.
template <int NSUB, int MODE>
__device__ __forceinline__ void fwd_epi_tile(const TcFwd &p, int row0, int ct0, uint32_t tacc,
                                             int nx, float *tile_s, float *wx_s,
                                             const float *xs_s, uint64_t *drained, int eg = 0) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int e = (warp - 2) & 7, q = warp & 3, hh = e >> 2;
  const int et = e * 32 + lane;  // 0..255
  const int H = p.H;
#pragma unroll 1
  for (int sub = 0; sub < NSUB; ++sub) {
    const int ct = ct0 + sub;
    // ---- phase 1: TMEM -> smem tile (thread = one accumulator row, 32 of the 64 columns)
    if (sub > 0) epi_bar(eg);  // previous sub-tile done reading tile_s / wx_s
    {
      const int r = q * 32 + lane;
      float acc[32];
      if (p.nkb) {
        const uint32_t taddr = tacc + (uint32_t(q * 32) << 16) + sub * 64 + hh * 32;
        tmem_ld16(taddr, acc);
        tmem_ld16(taddr + 16, acc + 16);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = 0.f;
      }
      float *dst = tile_s + r * kTileLd + hh * 32;
#pragma unroll
      for (int i = 0; i < 32; i += 4) st4(dst + i, make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]));
    }
    if (sub > 0)  // x-part weight rows of this sub-tile
      for (int i = et; i < nx * 64; i += kEpiThreads) {
        const int mf = i / 64, j = i % 64, m = mf / p.F, f = mf % p.F;
        wx_s[i] = __ldg(p.Wx + int64_t(m * p.C_in + f) * p.Nout + ct * 64 + j);
      }
    if (drained && sub == NSUB - 1) tc_fence_before();  // every TMEM load of the tile is done
    epi_bar(eg);
    if (drained && sub == NSUB - 1 && et == 0) mbar_arrive(drained);  // accumulator reusable
    // ---- phase 2: coalesced element-wise epilogue: 16 threads per row, 4 columns each
#pragma unroll 2
    for (int it = 0; it < (kBM * 64 / 4) / kEpiThreads; ++it) {
      const int idx = it * kEpiThreads + et;
      const int rl = idx >> 4, c4 = (idx & 15) * 4;
      const int row = row0 + rl;
      const bool valid = row < p.R;
      float4 a = ld4(tile_s + rl * kTileLd + c4);
      if (MODE == kEpiBwd) {
        if (!valid) continue;
        if (ct == p.fuse_tile) {
          // fused gate backward: a = d(r*H_{t-1}); dG_r = a H r (1-r); dH_{t-1} += a r
          const int64_t ro = int64_t(row) * 64 + c4, rg = int64_t(row) * 128 + c4;
          const float4 hp = ld4(p.Hprev + ro), rr = ld4_bf16(p.g_r + ro), dh = ld4(p.g_dHprev + ro);
          const float4 g = make_float4(a.x * hp.x * rr.x * (1.f - rr.x), a.y * hp.y * rr.y * (1.f - rr.y),
                                       a.z * hp.z * rr.z * (1.f - rr.z), a.w * hp.w * rr.w * (1.f - rr.w));
          st4(p.g_dHprev + ro, make_float4(fmaf(a.x, rr.x, dh.x), fmaf(a.y, rr.y, dh.y),
                                           fmaf(a.z, rr.z, dh.z), fmaf(a.w, rr.w, dh.w)));
          if (p.g_dG) st4(p.g_dG + rg, g);
          st4_bf16(p.g_dGb + rg, g);
        } else {
          float *d = p.dst[ct] + int64_t(row) * 64 + c4;
          if (p.dst_acc[ct]) {
            const float4 o = ld4(d);
            a.x += o.x, a.y += o.y, a.z += o.z, a.w += o.w;
          }
          st4(d, a);
        }
        continue;
      }
      // forward: pre-activation = acc + bias (+ layer-0 x part)
      const int jg = ct * 64 + c4;
      const float4 b = ld4(p.bias + jg);
      a.x += b.x, a.y += b.y, a.z += b.z, a.w += b.w;
      if (nx) {
        const float *xr = xs_s + rl * nx;
        for (int mf = 0; mf < nx; ++mf) {
          const float xv = xr[mf];
          const float4 w = ld4(wx_s + mf * 64 + c4);
          a.x = fmaf(xv, w.x, a.x), a.y = fmaf(xv, w.y, a.y);
          a.z = fmaf(xv, w.z, a.z), a.w = fmaf(xv, w.w, a.w);
        }
      }
      const int jh = (MODE == kEpiGate ? 0 : ct * 64) + c4;  // hidden unit of column c4
      const int64_t ro = int64_t(row) * H + jh;
      if (MODE == kEpiGate) {
        const float4 s = p.exact ? make_float4(sigmoid_f(a.x), sigmoid_f(a.y), sigmoid_f(a.z), sigmoid_f(a.w))
                                 : make_float4(sigmoid_mufu(a.x), sigmoid_mufu(a.y),
                                               sigmoid_mufu(a.z), sigmoid_mufu(a.w));
        if (valid) {
          if (ct == 0) {
            st4_bf16(p.out_r + ro, s);
            float4 hp = make_float4(0.f, 0.f, 0.f, 0.f);
            if (p.Hprev) hp = ld4(p.Hprev + ro);
            st4_bf16(p.out_rH + ro, make_float4(s.x * hp.x, s.y * hp.y, s.z * hp.z, s.w * hp.w));
          } else {
            st4(p.out_u + ro, s);
          }
        }
      } else {  // kEpiCand
        float4 hn = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid) {
          const float4 c = p.exact ? make_float4(tanhf(a.x), tanhf(a.y), tanhf(a.z), tanhf(a.w))
                                   : make_float4(tanh_mufu(a.x), tanh_mufu(a.y), tanh_mufu(a.z),
                                                 tanh_mufu(a.w));
          const float4 u = ld4(p.u_in + ro);
          float4 hp = make_float4(0.f, 0.f, 0.f, 0.f);
          if (p.Hprev) hp = ld4(p.Hprev + ro);
          hn = make_float4(u.x * hp.x + (1.f - u.x) * c.x, u.y * hp.y + (1.f - u.y) * c.y,
                           u.z * hp.z + (1.f - u.z) * c.z, u.w * hp.w + (1.f - u.w) * c.w);
          st4_bf16(p.out_c + ro, c);
          st4(p.out_H + ro, hn);
          st4_bf16(p.out_Hb + ro, hn);
        }
        if (p.yhat) {  // readout: 16 lanes of this row hold its 64 hidden units
#pragma unroll
          for (int o = 0; o < 4; ++o) {
            if (o >= p.F_out) break;
            float y = hn.x * __ldg(p.Wout + (jh + 0) * p.F_out + o) +
                      hn.y * __ldg(p.Wout + (jh + 1) * p.F_out + o) +
                      hn.z * __ldg(p.Wout + (jh + 2) * p.F_out + o) +
                      hn.w * __ldg(p.Wout + (jh + 3) * p.F_out + o);
#pragma unroll
            for (int off = 8; off > 0; off >>= 1) y += __shfl_xor_sync(0xffffffffu, y, off);
            if ((lane & 15) == 0 && valid)
              p.yhat[int64_t(row) * p.F_out + o] = y + __ldg(p.bout + o);
          }
        }
      }
    }
  }
}

// NSUB = 64-column sub-tiles per CTA: 1 (small R: more CTAs) or 2 (large R: A read once for
// both the r and u halves of the gate / the input and hidden tiles of the backward GEMM).
// MODE (kEpiGate / kEpiCand / kEpiBwd) is compile-time so each epilogue gets its own registers.
template <int NSUB, int MODE>
__global__ void __launch_bounds__(kFwdThreads, 2)
    k_tc_fwd(const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
             const __grid_constant__ CUtensorMap mB, const __grid_constant__ TcFwd p) {
  constexpr int NT = 64 * NSUB;
  constexpr int A_BYTES = kBM * kBK * 2, B_BYTES = NT * kBK * 2, STAGE = A_BYTES + B_BYTES;
  constexpr int kStages = fwd_stages(NSUB);  // two CTAs per SM: one's epilogue overlaps the
                                             // other's main loop
  static_assert(kStages * STAGE >= kBM * kTileLd * 4, "epilogue tile reuses the stage buffers");
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = align1024(smem_raw);
  Barriers *bar = carve<A_BYTES, B_BYTES, kStages>(smem);
  float *wx_s = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(bar) + 256);  // [20][64]
  float *tile_s = reinterpret_cast<float *>(smem);                                  // [128][68]
  float *xs_s = wx_s + 20 * 64;  // [128][<=20]: own region, filled while the MMAs run
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int row0 = blockIdx.x * kBM, ct0 = blockIdx.y * NSUB;
  griddep_launch_dependents();
  if (threadIdx.x == 0) tma_prefetch(&mA0), tma_prefetch(&mA1), tma_prefetch(&mB);
  setup(bar, NT);  // barriers + TMEM: the prologue that may overlap the predecessor's tail
  const uint32_t tmem = bar->tmem;

  if (warp == 0) {
    if (lane == 0) {
      // The weight tiles (B) were written by a plain (non-PDL) launch at the start of the step,
      // which completed before any later kernel started: the first ring's B loads go out before
      // griddepcontrol.wait, the A loads (the predecessor's outputs) after it.
      const int pre = min(p.nkb, kStages);
      for (int kb = 0; kb < pre; ++kb) {
        mbar_expect_tx(&bar->full[kb], STAGE);
        tma_load_3d(smem + kb * STAGE + A_BYTES, &mB, &bar->full[kb], p.kb_bx[kb],
                    p.kb_by[kb] + ct0 * 64, p.kb_bz[kb]);
      }
      griddep_wait();
      for (int kb = 0; kb < p.nkb; ++kb) {
        const int s = kb % kStages;
        uint8_t *a = smem + s * STAGE;
        if (kb >= pre) {
          mbar_wait(&bar->empty[s], ((kb / kStages) & 1) ^ 1);
          mbar_expect_tx(&bar->full[s], STAGE);
          tma_load_3d(a + A_BYTES, &mB, &bar->full[s], p.kb_bx[kb], p.kb_by[kb] + ct0 * 64,
                      p.kb_bz[kb]);
        }
        tma_load_3d(a, p.kb_as[kb] ? &mA1 : &mA0, &bar->full[s], p.kb_ac[kb], row0, p.kb_am[kb]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(kBM, NT, false, false);
      for (int kb = 0; kb < p.nkb; ++kb) {
        const int s = kb % kStages;
        mbar_wait(&bar->full[s], (kb / kStages) & 1);
        tc_fence_after();
        const uint32_t a = smem_u32(smem + s * STAGE), b = a + A_BYTES;
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)
          mma_bf16(tmem, desc_sw128(a + 32 * k, 16, 1024), desc_sw128(b + 32 * k, 16, 1024), idesc,
                   (kb | k) != 0);
        mma_commit(&bar->empty[s]);
      }
      mma_commit(&bar->tfull);
    }
  } else {
    griddep_wait();  // the epilogue reads the predecessor's outputs (H_{t-1}, u, r, dH, ...)
    const int et = (warp - 2) * 32 + lane;
    const int nx = fwd_epi_prepare<NSUB, MODE>(p, row0, ct0, et, wx_s, xs_s);
    mbar_wait(&bar->tfull, 0);  // MMAs done => every stage buffer is free for the tile
    tc_fence_after();
    fwd_epi_tile<NSUB, MODE>(p, row0, ct0, tmem, nx, tile_s, wx_s, xs_s, nullptr);
  }
  teardown(bar, NT);
}

// ------------------------------------------------------------------ persistent forward GEMM
// The same GEMM and epilogue as k_tc_fwd, as one persistent CTA per SM with TWO epilogue groups
// of 8 warps and a double-buffered TMEM accumulator: the CTA walks the (row tile, column tile)
// pairs t = blockIdx.x + i gridDim.x; tile i accumulates into TMEM buffer i & 1 and is drained
// by epilogue group i & 1 (its own shared tile and named barrier), so the TMA producer and the
// MMA warp run ahead into the next tile while the two groups drain the previous two -- the
// overlap two co-resident CTAs give, without the producer ever stopping for an epilogue.
// (A single epilogue group measured slower than two CTAs per SM: the fused GRU epilogue, not the
// main loop, bounds these GEMMs.)  PGTI_TC_PERSIST=0 selects the per-tile kernel.
constexpr int kStagesP = 3, kFwdpThreads = 64 + 2 * kEpiThreads;
struct BarriersP {
  uint64_t full[kStagesP], empty[kStagesP], tfull[2], tempty[2];
  uint32_t tmem;
};
constexpr int kEpiRegionBytes = kBM * kTileLd * 4 + 20 * 64 * 4 + kBM * 20 * 4;
constexpr int fwdp_smem_bytes(int nsub) {
  return kStagesP * (kBM * kBK * 2 + 64 * nsub * kBK * 2) + 2 * kEpiRegionBytes +
         int(sizeof(BarriersP)) + 1024 + 64;
}

template <int NSUB, int MODE>
__global__ void __launch_bounds__(kFwdpThreads, 1)
    k_tc_fwdp(const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
              const __grid_constant__ CUtensorMap mB, const __grid_constant__ TcFwd p,
              int ncol_tiles, int ntiles) {
  constexpr int NT = 64 * NSUB;
  constexpr int A_BYTES = kBM * kBK * 2, B_BYTES = NT * kBK * 2, STAGE = A_BYTES + B_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = align1024(smem_raw);
  uint8_t *epi = smem + kStagesP * STAGE;  // [2][tile_s 128x68 | wx_s 20x64 | xs_s 128x20]
  BarriersP *bar = reinterpret_cast<BarriersP *>(epi + 2 * kEpiRegionBytes);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  griddep_launch_dependents();
  if (threadIdx.x == 0) {
    tma_prefetch(&mA0), tma_prefetch(&mA1), tma_prefetch(&mB);
    for (int s = 0; s < kStagesP; ++s) mbar_init(&bar->full[s], 1), mbar_init(&bar->empty[s], 1);
    for (int a = 0; a < 2; ++a) mbar_init(&bar->tfull[a], 1), mbar_init(&bar->tempty[a], 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&bar->tmem, 2 * NT);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar->tmem;

  if (warp == 0) {
    if (lane == 0) {
      // weight tiles (B) come from a plain launch earlier in the step: the first tile's first
      // ring of B loads goes out before griddepcontrol.wait, everything else after it
      int g = 0;  // k-blocks issued so far (position in the stage ring)
      const int pre = min(p.nkb, kStagesP);
      {
        const int ct0 = (int(blockIdx.x) % ncol_tiles) * NSUB;
        for (int kb = 0; kb < pre; ++kb) {
          mbar_expect_tx(&bar->full[kb], STAGE);
          tma_load_3d(smem + kb * STAGE + A_BYTES, &mB, &bar->full[kb], p.kb_bx[kb],
                      p.kb_by[kb] + ct0 * 64, p.kb_bz[kb]);
        }
      }
      griddep_wait();
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int row0 = (t / ncol_tiles) * kBM, ct0 = (t % ncol_tiles) * NSUB;
        for (int kb = 0; kb < p.nkb; ++kb, ++g) {
          const int s = g % kStagesP;
          uint8_t *a = smem + s * STAGE;
          if (g >= pre) {
            if (g >= kStagesP) mbar_wait(&bar->empty[s], ((g / kStagesP) & 1) ^ 1);
            mbar_expect_tx(&bar->full[s], STAGE);
            tma_load_3d(a + A_BYTES, &mB, &bar->full[s], p.kb_bx[kb], p.kb_by[kb] + ct0 * 64,
                        p.kb_bz[kb]);
          }
          tma_load_3d(a, p.kb_as[kb] ? &mA1 : &mA0, &bar->full[s], p.kb_ac[kb], row0,
                      p.kb_am[kb]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(kBM, NT, false, false);
      int g = 0, i = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int ab = i & 1;
        if (i >= 2) {  // group ab has drained this accumulator's previous tile
          mbar_wait(&bar->tempty[ab], ((i >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        const uint32_t tacc = tmem + uint32_t(ab * NT);
        for (int kb = 0; kb < p.nkb; ++kb, ++g) {
          const int s = g % kStagesP;
          mbar_wait(&bar->full[s], (g / kStagesP) & 1);
          tc_fence_after();
          const uint32_t a = smem_u32(smem + s * STAGE), b = a + A_BYTES;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            mma_bf16(tacc, desc_sw128(a + 32 * k, 16, 1024), desc_sw128(b + 32 * k, 16, 1024),
                     idesc, (kb | k) != 0);
          mma_commit(&bar->empty[s]);
        }
        mma_commit(&bar->tfull[ab]);
      }
    }
  } else {
    griddep_wait();  // the epilogue reads the predecessor's outputs (H_{t-1}, u, r, dH, ...)
    const int eg = (warp - 2) >> 3;  // epilogue group: tiles i with i & 1 == eg
    const int et = ((warp - 2) & 7) * 32 + lane;
    float *tile_s = reinterpret_cast<float *>(epi + eg * kEpiRegionBytes);
    float *wx_s = tile_s + kBM * kTileLd;
    float *xs_s = wx_s + 20 * 64;
    int k = 0;  // this group's tiles so far
    for (int t = blockIdx.x + eg * gridDim.x; t < ntiles; t += 2 * gridDim.x, ++k) {
      const int row0 = (t / ncol_tiles) * kBM, ct0 = (t % ncol_tiles) * NSUB;
      if (k > 0) epi_bar(eg);  // the previous tile's phase 2 is done with tile_s / wx_s / xs_s
      const int nx = fwd_epi_prepare<NSUB, MODE>(p, row0, ct0, et, wx_s, xs_s);
      mbar_wait(&bar->tfull[eg], k & 1);
      tc_fence_after();
      fwd_epi_tile<NSUB, MODE>(p, row0, ct0, tmem + uint32_t(eg * NT), nx, tile_s, wx_s, xs_s,
                               &bar->tempty[eg], eg);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 2 * NT);
  }
}

// ================================================================== wgrad (MN-major A and B)
constexpr int kWgThreads = 192;

// Split-K plan of the weight gradient.  The reduction dimension is the (t, row) index space,
// walked as k-steps of kBK rows that never cross a time step: k-step ks covers rows
// [(ks % nrb) kBK, +kBK) of step t = ks / nrb (nrb = ceil(R / kBK); rows >= R are TMA zero
// fill).  The T nrb k-steps are cut into `nchunks` contiguous ranges, one CTA per (v tile,
// range), so the grid is about one wave of the 148 SMs at any R (one CTA per SM: 128 KB of
// stages) and each CTA accumulates its whole range in TMEM: at full PeMS 29 partial tiles per
// output instead of 12 x 349, i.e. ~20 MB of partials instead of 1.4 GB.
struct WgPlan {
  int nrb;       // k-steps per time step
  int total;     // T * nrb
  int nchunks;   // contiguous k-step ranges (split-K factor)
};

WgPlan wg_plan(int V, int T, int R) {
  WgPlan q;
  q.nrb = int(ceil_div(R, kBK));
  q.total = T * q.nrb;
  const int tiles = int(ceil_div(V, kBM));
  q.nchunks = std::max(1, std::min(q.total, kNumSMs / tiles));
  return q;
}

template <int NOUT>
__global__ void __launch_bounds__(kWgThreads, 1)
    k_tc_wgrad(const __grid_constant__ CUtensorMap mA_in, const __grid_constant__ CUtensorMap mA_h,
               const __grid_constant__ CUtensorMap mG, const __grid_constant__ TcWgrad p,
               WgPlan q) {
  constexpr int A_BYTES = kBM * kBK * 2, B_BYTES = NOUT * kBK * 2, STAGE = A_BYTES + B_BYTES;
  constexpr int NCH_B = NOUT / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = align1024(smem_raw);
  Barriers *bar = carve<A_BYTES, B_BYTES>(smem);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tile = blockIdx.x, chunk = blockIdx.y;
  // k-steps [ks0, ks1) of this chunk: an even split of the T nrb k-steps (fixed, so the
  // partials and their fixed-order reduction are bitwise reproducible)
  const int ks0 = int(int64_t(q.total) * chunk / q.nchunks);
  const int ks1 = int(int64_t(q.total) * (chunk + 1) / q.nchunks);
  const int nst = ks1 - ks0;
  griddep_launch_dependents();
  if (threadIdx.x == 0) tma_prefetch(&mA_in), tma_prefetch(&mA_h), tma_prefetch(&mG);
  setup(bar, NOUT);  // barriers + TMEM while the predecessor drains
  griddep_wait();    // every operand is a predecessor's output
  const uint32_t tmem = bar->tmem;
  if (warp == 0) {
    if (lane == 0)
      for (int st = 0, t = ks0 / q.nrb, rb = ks0 - t * q.nrb; st < nst; ++st) {
        const int s = st % kStages, row = rb * kBK;
        mbar_wait(&bar->empty[s], ((st / kStages) & 1) ^ 1);
        mbar_expect_tx(&bar->full[s], STAGE);
        uint8_t *a = smem + s * STAGE;
#pragma unroll
        for (int qc = 0; qc < 2; ++qc) {
          // chunk qc of this 128-row v tile -> (source, block m)
          int src, m;
          if (p.vseg == 128) src = qc, m = tile;
          else src = 1, m = 2 * tile + qc;
          if (p.x_F && m == p.M) src = 0, m = 0;  // layer 0: the packed input rows
          const int tt = src ? t + p.h_toff : t;     // tt < 0 or m >= M -> TMA zero fill
          tma_load_4d(a + qc * (A_BYTES / 2), src ? &mA_h : &mA_in, &bar->full[s], 0, row, m, tt);
        }
#pragma unroll
        for (int qc = 0; qc < NCH_B; ++qc)
          tma_load_3d(a + A_BYTES + qc * 8192, &mG, &bar->full[s], qc * 64, row, t);
        if (++rb == q.nrb) rb = 0, ++t;
      }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(kBM, NOUT, true, true);
      for (int st = 0; st < nst; ++st) {
        const int s = st % kStages;
        mbar_wait(&bar->full[s], (st / kStages) & 1);
        tc_fence_after();
        const uint32_t a = smem_u32(smem + s * STAGE), b = a + A_BYTES;
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)
          mma_bf16(tmem, desc_sw128(a + 2048 * k, 8192, 1024), desc_sw128(b + 2048 * k, 8192, 1024),
                   idesc, (st | k) != 0);
        mma_commit(&bar->empty[s]);
      }
      mma_commit(&bar->tfull);
    }
  } else {
    const int q = warp & 3;
    const int v = tile * kBM + q * 32 + lane;
    const uint32_t taddr = tmem + (uint32_t(q * 32) << 16);
    mbar_wait(&bar->tfull, 0);
    tc_fence_after();
    float *out = p.partial + (int64_t(chunk) * p.V + v) * NOUT;
    for (int c0 = 0; c0 < NOUT; c0 += 16) {
      float d[16];
      tmem_ld16(taddr + c0, d);
      tmem_wait_ld();
      if (v >= p.V) continue;
      if (nst == 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) d[i] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < 16; i += 4)
        *reinterpret_cast<float4 *>(out + c0 + i) = make_float4(d[i], d[i + 1], d[i + 2], d[i + 3]);
    }
  }
  teardown(bar, NOUT);
}

__global__ void k_tc_reduce(const float *__restrict__ partial, int nchunks, int V, int Nout,
                            int vseg, int coff, int C_in, int M, int x_F, int x_bias,
                            float *__restrict__ out) {
  griddep_launch_dependents();
  griddep_wait();
  const int64_t n = int64_t(V) * Nout;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    // chunks summed in index order (bitwise reproducible); eight loads in flight per batch
    float s = 0.f;
    int c = 0;
    for (; c + 8 <= nchunks; c += 8) {
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldg(partial + int64_t(c + k) * n + i);
#pragma unroll
      for (int k = 0; k < 8; ++k) s += v[k];
    }
    for (; c < nchunks; ++c) s += __ldg(partial + int64_t(c) * n + i);
    const int v = int(i / Nout), j = int(i - int64_t(v) * Nout);
    const int m = v / vseg;
    if (x_F && m == M) {  // packed input channel c = m' x_F + f -> row m' C_in + f
      const int c = v - m * vseg, mm = c / x_F, f = c - mm * x_F;
      if (c < M * x_F) out[int64_t(mm * C_in + f) * Nout + j] = s;
      else if (x_bias && c == M * x_F) out[int64_t(M * C_in) * Nout + j] = s;  // sum of dG
      continue;
    }
    out[int64_t(m * C_in + coff + (v - m * vseg)) * Nout + j] = s;
  }
}

// ================================================================== host side
PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// bf16 tensor map, SWIZZLE_128B, zero OOB fill.  dims[0] is the contiguous dimension.
bool make_map(CUtensorMap *m, const void *base, int rank, const uint64_t *dims,
              const uint64_t *strides_bytes, const uint32_t *box) {
  std::memset(m, 0, sizeof(*m));
  if (!base) return true;  // unused operand
  auto enc = encoder();
  if (!enc) return false;
  const uint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void *>(base), dims,
                   strides_bytes, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <typename K>
cudaError_t set_smem(K kernel, int bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

constexpr int wg_smem_bytes(int b_rows) { return kStages * (kBM * kBK * 2 + b_rows * kBK * 2) + 1024 + 256; }
constexpr int fwd_smem_bytes(int nsub) {
  return fwd_stages(nsub) * (kBM * kBK * 2 + 64 * nsub * kBK * 2) + 1024 + 256 + 20 * 64 * 4 +
         kBM * 20 * 4;
}

}  // namespace

cudaError_t launch_tc_fwd(const TcFwd &p_in, cudaStream_t s) {
  TcFwd p = p_in;
  {  // gate / candidate activations by the MUFU tanh (bf16 path); PGTI_TC_EXACT=1: libm forms
    const char *e = std::getenv("PGTI_TC_EXACT");
    p.exact = (e && e[0] == '1') ? 1 : 0;
  }
  if (p.H != 64 || p.nkb > kTcMaxKb || (p.Dx && p.F * p.M > 20) || p.F_out > 4 ||
      p.ntiles < 1 || p.ntiles > 2 || (p.CA != 64 && p.CA != 128))
    return cudaErrorInvalidValue;
  CUtensorMap ma0, ma1, mb;
  const uint64_t R = uint64_t(p.R), CA = uint64_t(p.CA);
  const uint64_t dA0[3] = {CA, R, uint64_t(p.M0)}, dA1[3] = {CA, R, uint64_t(p.M1)};
  const uint64_t sA[2] = {CA * 2, R * CA * 2};
  const uint32_t bA[3] = {64, 128, 1};
  const uint64_t dB[3] = {uint64_t(p.bX), uint64_t(p.bY), uint64_t(p.bZ)},
                 sB[2] = {uint64_t(p.bX) * 2, uint64_t(p.bX) * p.bY * 2};
  // two 64-column sub-tiles per CTA once there are enough row tiles to fill the GPU twice:
  // A (the dominant operand) is then staged once for both halves
  const int row_tiles = int(ceil_div(p.R, kBM));
  const int nsub = (p.ntiles == 2 && row_tiles >= 2 * kNumSMs) ? 2 : 1;
  const uint32_t bB[3] = {64, uint32_t(64 * nsub), 1};
  if (!make_map(&ma0, p.A0, 3, dA0, sA, bA) || !make_map(&ma1, p.A1, 3, dA1, sA, bA) ||
      !make_map(&mb, p.Bw, 3, dB, sB, bB))
    return cudaErrorInvalidValue;
  const dim3 grid(unsigned(row_tiles), unsigned(p.ntiles / nsub));
  const double N = 64.0 * p.ntiles;
  const double Kt = double(p.nkb) * 64 + (p.Dx ? p.F * p.M : 0);
  double io = p.mode == kEpiGate ? 2 + (p.Hprev ? 1 : 0) + 0.5
            : p.mode == kEpiCand ? 4.5 + (p.Hprev ? 1 : 0)
                                 : 1.0 + (p.dst_acc[0] ? 1.0 : 0.0);
  const double bytes = 2.0 * p.R * 64 * p.nkb + 2.0 * p.nkb * 64 * N + 4.0 * p.R * N * io / 2 * 2;
  ProfScope prof(p.mode == kEpiBwd ? kProfGemmDgrad : kProfGemmFwd, s, bytes, 2.0 * p.R * Kt * N);
  static const bool persist = [] {
    const char *e = std::getenv("PGTI_TC_PERSIST");
    return !(e && e[0] == '0');
  }();
  // persistent form once every SM gets >= 4 tiles (full PeMS: 5,580; PeMS-All-LA: 1,358): full
  // PeMS 883 -> 930 samples/s; with few tiles per SM (METR-LA: 208) the per-tile kernel with two
  // CTAs per SM is faster (39.8 K vs 35.6 K)
  const int ncol = p.ntiles / nsub, ntiles = row_tiles * ncol;
  if (persist && p.nkb > 0 && ntiles >= 4 * kNumSMs) {
    const int gridp = std::min(ntiles, kNumSMs);
    const int smem = fwdp_smem_bytes(nsub);
    auto gop = [&](auto kernel) -> cudaError_t {
      cudaError_t e = set_smem(kernel, smem);
      if (e != cudaSuccess) return e;
      return pdl_launch(kernel, dim3(unsigned(gridp)), dim3(kFwdpThreads), smem, s, ma0, ma1,
                        mb, p, ncol, ntiles);
    };
    switch (p.mode * 2 + (nsub - 1)) {
      case kEpiGate * 2: return gop(k_tc_fwdp<1, kEpiGate>);
      case kEpiGate * 2 + 1: return gop(k_tc_fwdp<2, kEpiGate>);
      case kEpiCand * 2: return gop(k_tc_fwdp<1, kEpiCand>);
      case kEpiCand * 2 + 1: return gop(k_tc_fwdp<2, kEpiCand>);
      case kEpiBwd * 2: return gop(k_tc_fwdp<1, kEpiBwd>);
      case kEpiBwd * 2 + 1: return gop(k_tc_fwdp<2, kEpiBwd>);
      default: return cudaErrorInvalidValue;
    }
  }
  auto go = [&](auto kernel, int smem) -> cudaError_t {
    cudaError_t e = set_smem(kernel, smem);  // idempotent, cheap
    if (e != cudaSuccess) return e;
    return pdl_launch(kernel, grid, dim3(kFwdThreads), smem, s, ma0, ma1, mb, p);
  };
  const int sm1 = fwd_smem_bytes(1), sm2 = fwd_smem_bytes(2);
  switch (p.mode * 2 + (nsub - 1)) {
    case kEpiGate * 2: return go(k_tc_fwd<1, kEpiGate>, sm1);
    case kEpiGate * 2 + 1: return go(k_tc_fwd<2, kEpiGate>, sm2);
    case kEpiCand * 2: return go(k_tc_fwd<1, kEpiCand>, sm1);
    case kEpiCand * 2 + 1: return go(k_tc_fwd<2, kEpiCand>, sm2);
    case kEpiBwd * 2: return go(k_tc_fwd<1, kEpiBwd>, sm1);
    case kEpiBwd * 2 + 1: return go(k_tc_fwd<2, kEpiBwd>, sm2);
    default: return cudaErrorInvalidValue;
  }
}

size_t tc_wgrad_partial_floats(int V, int Nout, int T, int R) {
  return size_t(wg_plan(V, T, R).nchunks) * size_t(V) * size_t(Nout);
}

cudaError_t launch_tc_wgrad(const TcWgrad &p, cudaStream_t s) {
  if ((p.Nout != 128 && p.Nout != 64) || (p.vseg != 64 && p.vseg != 128)) return cudaErrorInvalidValue;
  CUtensorMap ma_in, ma_h, mg;
  const uint64_t R = uint64_t(p.R), M = uint64_t(p.M), T = uint64_t(p.T);
  const uint64_t dA[4] = {64, R, M, T}, sA[3] = {128, R * 128, M * R * 128};
  const uint32_t bA[4] = {64, 64, 1, 1};
  const uint64_t dG[3] = {uint64_t(p.Nout), R, T}, sG[2] = {uint64_t(p.Nout) * 2, R * p.Nout * 2};
  const uint32_t bG[3] = {64, 64, 1};
  if (p.x_F && (p.vseg != 64 || p.V != (p.M + 1) * 64 || !p.A_in)) return cudaErrorInvalidValue;
  // A_in is [T][M][R][64] (layer > 0) or, with x_F, the packed input rows [T][1][R][64]
  const uint64_t Min = p.x_F ? 1 : M;
  const uint64_t dAi[4] = {64, R, Min, T}, sAi[3] = {128, R * 128, Min * R * 128};
  if (!make_map(&ma_in, p.A_in, 4, dAi, sAi, bA) || !make_map(&ma_h, p.A_h, 4, dA, sA, bA) ||
      !make_map(&mg, p.G, 3, dG, sG, bG))
    return cudaErrorInvalidValue;
  const WgPlan q = wg_plan(p.V, p.T, p.R);
  const int nchunks = q.nchunks;
  if (int64_t(nchunks) * p.V * p.Nout > p.partial_cap) return cudaErrorInvalidValue;
  const dim3 grid(unsigned(ceil_div(p.V, kBM)), unsigned(nchunks));
  const int64_t n = int64_t(p.V) * p.Nout;
  cudaError_t e;
  {
    const double TR = double(p.T) * p.R;
    ProfScope prof(kProfGemmWgrad, s, 2.0 * TR * p.V + 2.0 * TR * p.Nout + 4.0 * nchunks * n,
                   2.0 * TR * p.V * p.Nout);
    // the >48 KB opt-in is per device: set on every launch (cheap), as launch_tc_fwd does
    if (p.Nout == 128) {
      e = set_smem(k_tc_wgrad<128>, wg_smem_bytes(128));
      if (e != cudaSuccess) return e;
      e = pdl_launch(k_tc_wgrad<128>, grid, dim3(kWgThreads), wg_smem_bytes(128), s, ma_in, ma_h,
                     mg, p, q);
    } else {
      e = set_smem(k_tc_wgrad<64>, wg_smem_bytes(64));
      if (e != cudaSuccess) return e;
      e = pdl_launch(k_tc_wgrad<64>, grid, dim3(kWgThreads), wg_smem_bytes(64), s, ma_in, ma_h,
                     mg, p, q);
    }
  }
  if (e != cudaSuccess) return e;
  ProfScope prof(kProfReduce, s, 4.0 * double(n) * (nchunks + 1), double(n) * nchunks);
  return pdl_launch(k_tc_reduce, dim3(unsigned(std::min<int64_t>(ceil_div(n, 256), 1184))),
                    dim3(256), 0, s, static_cast<const float *>(p.partial), nchunks, p.V, p.Nout,
                    p.vseg, p.coff, p.C_in, p.M, p.x_F, p.x_bias, p.out);
}

}  // namespace pgti
