// K3: tcgen05 gate GEMMs (bf16 operands staged by TMA into SWIZZLE_128B shared memory, fp32
// accumulators in TMEM, one elected thread issuing tcgen05.mma) with the GRU math fused into
// the TMEM -> register epilogue.
//   k_tc_fwd   : multi-block GEMM (forward gates, and the backward "diffuse-then-GEMM" dgrad)
//                10 warps: warp 0 TMA producer, warp 1 TMEM alloc + MMA issuer, warps 2-9
//                epilogue (thread = one accumulator row x 32 of the tile's 64 columns)
//   k_tc_wgrad : split-K weight gradient, MN-major A (diffusion blocks) and B (gate gradients)
// 4-stage mbarrier ring between TMA and MMA (full / empty), one commit barrier MMA -> epilogue.
// Equations: Li et al. Eq. 2-3 [ext], PAPER.md P:168, P:222 (readings c1-c7).
#include <cudaTypedefs.h>

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

template <int A_BYTES, int B_BYTES>
__device__ __forceinline__ Barriers *carve(uint8_t *smem) {
  return reinterpret_cast<Barriers *>(smem + kStages * (A_BYTES + B_BYTES));
}

__device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
  return reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
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

// ================================================================== multi-block GEMM
// One CTA = 128 rows x one 64-column tile.  Everything the epilogue needs that does not depend
// on the accumulator (bias, layer-0 x part by FFMA, H_{t-1}, u, the bwd destination) is
// gathered while the MMAs run; after the commit barrier only TMEM -> math -> stores remain.
constexpr int kFwdThreads = 320, kEpiThreads = 256;

__device__ __forceinline__ void epi_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
}

// NSUB = 64-column sub-tiles per CTA: 1 (small R: more CTAs) or 2 (large R: A read once for
// both the r and u halves of the gate / the input and hidden tiles of the backward GEMM).
template <int NSUB>
__global__ void __launch_bounds__(kFwdThreads, 3 - NSUB)
    k_tc_fwd(const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
             const __grid_constant__ CUtensorMap mB, const __grid_constant__ TcFwd p) {
  constexpr int NT = 64 * NSUB;
  constexpr int A_BYTES = kBM * kBK * 2, B_BYTES = NT * kBK * 2, STAGE = A_BYTES + B_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = align1024(smem_raw);
  Barriers *bar = carve<A_BYTES, B_BYTES>(smem);
  float *wx_s = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(bar) + 256);  // [20][64]
  float *y_s = wx_s + 20 * 64;                                                       // [128][4]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int row0 = blockIdx.x * kBM, ct0 = blockIdx.y * NSUB;
  if (threadIdx.x == 0) tma_prefetch(&mA0), tma_prefetch(&mA1), tma_prefetch(&mB);
  setup(bar, NT);
  const uint32_t tmem = bar->tmem;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < p.nkb; ++kb) {
        const int s = kb % kStages;
        mbar_wait(&bar->empty[s], ((kb / kStages) & 1) ^ 1);
        mbar_expect_tx(&bar->full[s], STAGE);
        uint8_t *a = smem + s * STAGE;
        tma_load_3d(a, p.kb_as[kb] ? &mA1 : &mA0, &bar->full[s], p.kb_ac[kb], row0, p.kb_am[kb]);
        tma_load_3d(a + A_BYTES, &mB, &bar->full[s], p.kb_bx[kb], p.kb_by[kb] + ct0 * 64,
                    p.kb_bz[kb]);
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
    const int e = warp - 2, q = warp & 3, hh = e >> 2;
    const int r = q * 32 + lane, row = row0 + r;
    const bool valid = row < p.R;
    const int H = p.H;
#pragma unroll 1
    for (int sub = 0; sub < NSUB; ++sub) {
    if (sub > 0) epi_bar();                  // sub-tile 0 finished with wx_s / y_s
    const int ct = ct0 + sub;
    const int jc = hh * 32;                  // first tile column of this thread
    const uint32_t tsub = uint32_t(sub * 64);  // TMEM column of this sub-tile
    if (p.mode == kEpiBwd) {
      float *dst = p.dst[ct];
      const int64_t ro = int64_t(row) * 64 + jc;
      float old[32];
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid && p.dst_acc[ct]) a = *reinterpret_cast<const float4 *>(dst + ro + i);
        old[i] = a.x, old[i + 1] = a.y, old[i + 2] = a.z, old[i + 3] = a.w;
      }
      mbar_wait(&bar->tfull, 0);
      tc_fence_after();
      float acc[32];
      const uint32_t taddr = tmem + (uint32_t(q * 32) << 16) + tsub + jc;
      tmem_ld16(taddr, acc);
      tmem_ld16(taddr + 16, acc + 16);
      tmem_wait_ld();
      if (valid) {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4 *>(dst + ro + i) =
              make_float4(old[i] + acc[i], old[i + 1] + acc[i + 1], old[i + 2] + acc[i + 2],
                          old[i + 3] + acc[i + 3]);
      }
    } else {
      const int nx = p.Dx ? p.F * p.M : 0;
      // stage this tile's x-part weight rows (fp32) in shared memory
      for (int i = e * 32 + lane; i < nx * 64; i += kEpiThreads) {
        const int mf = i / 64, j = i % 64, m = mf / p.F, f = mf % p.F;
        wx_s[i] = __ldg(p.Wx + int64_t(m * p.C_in + f) * p.Nout + ct * 64 + j);
      }
      epi_bar();
      const int jg = ct * 64 + jc;  // first gate column
      float pre[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) pre[i] = __ldg(p.bias + jg + i);
      if (nx && valid) {
        for (int mf = 0; mf < nx; ++mf) {
          const int m = mf / p.F, f = mf % p.F;
          const float xv = __ldg(p.Dx + m * p.dx_mstride + int64_t(row) * p.F + f);
#pragma unroll
          for (int i = 0; i < 32; ++i) pre[i] = fmaf(xv, wx_s[mf * 64 + jc + i], pre[i]);
        }
      }
      const int jh = (p.mode == kEpiGate ? 0 : ct * 64) + jc;  // hidden index of column 0
      const int64_t ro = int64_t(row) * H + jh;
      const bool need_h = p.mode == kEpiCand || ct == 0;
      float hp[32], uu[32];
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
        if (valid && need_h && p.Hprev) a = *reinterpret_cast<const float4 *>(p.Hprev + ro + i);
        if (valid && p.mode == kEpiCand) b = *reinterpret_cast<const float4 *>(p.u_in + ro + i);
        hp[i] = a.x, hp[i + 1] = a.y, hp[i + 2] = a.z, hp[i + 3] = a.w;
        uu[i] = b.x, uu[i + 1] = b.y, uu[i + 2] = b.z, uu[i + 3] = b.w;
      }
      mbar_wait(&bar->tfull, 0);
      tc_fence_after();
      float acc[32];
      if (p.nkb) {
        const uint32_t taddr = tmem + (uint32_t(q * 32) << 16) + tsub + jc;
        tmem_ld16(taddr, acc);
        tmem_ld16(taddr + 16, acc + 16);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = 0.f;
      }
      if (p.mode == kEpiGate) {
        float *out = ct == 0 ? p.out_r : p.out_u;
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = sigmoid_f(acc[i] + pre[i]);
        if (valid) {
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4 *>(out + ro + i) =
                make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
          if (ct == 0) {
#pragma unroll
            for (int i = 0; i < 32; ++i) hp[i] *= acc[i];
#pragma unroll
            for (int i = 0; i < 32; i += 8)
              *reinterpret_cast<uint4 *>(p.out_rH + ro + i) = pack8_bf16(hp + i);
          }
        }
      } else {
        float ys0 = 0.f, ys1 = 0.f, ys2 = 0.f, ys3 = 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float c = tanhf(acc[i] + pre[i]);
          acc[i] = c;
          pre[i] = uu[i] * hp[i] + (1.0f - uu[i]) * c;  // H_t
        }
        if (p.yhat) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float *w = p.Wout + (jh + i) * p.F_out;
            ys0 = fmaf(pre[i], __ldg(w), ys0);
            if (p.F_out > 1) ys1 = fmaf(pre[i], __ldg(w + 1), ys1);
            if (p.F_out > 2) ys2 = fmaf(pre[i], __ldg(w + 2), ys2);
            if (p.F_out > 3) ys3 = fmaf(pre[i], __ldg(w + 3), ys3);
          }
        }
        const float ys[4] = {ys0, ys1, ys2, ys3};
        if (valid) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            *reinterpret_cast<float4 *>(p.out_c + ro + i) = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
            *reinterpret_cast<float4 *>(p.out_H + ro + i) = make_float4(pre[i], pre[i + 1], pre[i + 2], pre[i + 3]);
          }
#pragma unroll
          for (int i = 0; i < 32; i += 8)
            *reinterpret_cast<uint4 *>(p.out_Hb + ro + i) = pack8_bf16(pre + i);
        }
        if (p.yhat) {
          if (hh == 1) {
#pragma unroll
            for (int o = 0; o < 4; ++o) y_s[r * 4 + o] = ys[o];
          }
          epi_bar();
          if (hh == 0 && valid) {
#pragma unroll
            for (int o = 0; o < 4; ++o)
              if (o < p.F_out)
                p.yhat[int64_t(row) * p.F_out + o] = (ys[o] + y_s[r * 4 + o]) + __ldg(p.bout + o);
          }
        }
      }
    }
    }  // sub-tiles
  }
  teardown(bar, NT);
}

// ================================================================== wgrad (MN-major A and B)
constexpr int kWgThreads = 192;
constexpr int kWKC = 2048;  // rows per split-K chunk

template <int NOUT>
__global__ void __launch_bounds__(kWgThreads, 1)
    k_tc_wgrad(const __grid_constant__ CUtensorMap mA_in, const __grid_constant__ CUtensorMap mA_h,
               const __grid_constant__ CUtensorMap mG, const __grid_constant__ TcWgrad p,
               int chunks_per_t) {
  constexpr int A_BYTES = kBM * kBK * 2, B_BYTES = NOUT * kBK * 2, STAGE = A_BYTES + B_BYTES;
  constexpr int NCH_B = NOUT / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = align1024(smem_raw);
  Barriers *bar = carve<A_BYTES, B_BYTES>(smem);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tile = blockIdx.x, chunk = blockIdx.y;
  const int t = chunk / chunks_per_t;
  const int rbeg = (chunk - t * chunks_per_t) * kWKC;
  const int rend = min(p.R, rbeg + kWKC);
  const int nst = (rend - rbeg + kBK - 1) / kBK;
  if (threadIdx.x == 0) tma_prefetch(&mA_in), tma_prefetch(&mA_h), tma_prefetch(&mG);
  setup(bar, NOUT);
  const uint32_t tmem = bar->tmem;
  if (warp == 0) {
    if (lane == 0)
      for (int st = 0; st < nst; ++st) {
        const int s = st % kStages, row = rbeg + st * kBK;
        mbar_wait(&bar->empty[s], ((st / kStages) & 1) ^ 1);
        mbar_expect_tx(&bar->full[s], STAGE);
        uint8_t *a = smem + s * STAGE;
#pragma unroll
        for (int qc = 0; qc < 2; ++qc) {
          // chunk qc of this 128-row v tile -> (source, block m)
          int src, m;
          if (p.vseg == 128) src = qc, m = tile;
          else src = 1, m = 2 * tile + qc;
          const int tt = src ? t + p.h_toff : t;     // tt < 0 or m >= M -> TMA zero fill
          tma_load_4d(a + qc * (A_BYTES / 2), src ? &mA_h : &mA_in, &bar->full[s], 0, row, m, tt);
        }
#pragma unroll
        for (int qc = 0; qc < NCH_B; ++qc)
          tma_load_3d(a + A_BYTES + qc * 8192, &mG, &bar->full[s], qc * 64, row, t);
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
                            int vseg, int coff, int C_in, float *__restrict__ out) {
  const int64_t n = int64_t(V) * Nout;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < nchunks; ++c) s += partial[int64_t(c) * n + i];
    const int v = int(i / Nout), j = int(i - int64_t(v) * Nout);
    const int m = v / vseg;
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
  return kStages * (kBM * kBK * 2 + 64 * nsub * kBK * 2) + 1024 + 256 + (20 * 64 + 128 * 4) * 4;
}

}  // namespace

cudaError_t launch_tc_fwd(const TcFwd &p, cudaStream_t s) {
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
  if (nsub == 2) {
    static cudaError_t once = set_smem(k_tc_fwd<2>, fwd_smem_bytes(2));
    if (once != cudaSuccess) return once;
    k_tc_fwd<2><<<grid, kFwdThreads, fwd_smem_bytes(2), s>>>(ma0, ma1, mb, p);
  } else {
    static cudaError_t once = set_smem(k_tc_fwd<1>, fwd_smem_bytes(1));
    if (once != cudaSuccess) return once;
    k_tc_fwd<1><<<grid, kFwdThreads, fwd_smem_bytes(1), s>>>(ma0, ma1, mb, p);
  }
  return cudaGetLastError();
}

size_t tc_wgrad_partial_floats(int V, int Nout, int T, int R) {
  return size_t(T) * size_t(ceil_div(R, kWKC)) * size_t(V) * size_t(Nout);
}

cudaError_t launch_tc_wgrad(const TcWgrad &p, cudaStream_t s) {
  if ((p.Nout != 128 && p.Nout != 64) || (p.vseg != 64 && p.vseg != 128)) return cudaErrorInvalidValue;
  CUtensorMap ma_in, ma_h, mg;
  const uint64_t R = uint64_t(p.R), M = uint64_t(p.M), T = uint64_t(p.T);
  const uint64_t dA[4] = {64, R, M, T}, sA[3] = {128, R * 128, M * R * 128};
  const uint32_t bA[4] = {64, 64, 1, 1};
  const uint64_t dG[3] = {uint64_t(p.Nout), R, T}, sG[2] = {uint64_t(p.Nout) * 2, R * p.Nout * 2};
  const uint32_t bG[3] = {64, 64, 1};
  if (!make_map(&ma_in, p.A_in, 4, dA, sA, bA) || !make_map(&ma_h, p.A_h, 4, dA, sA, bA) ||
      !make_map(&mg, p.G, 3, dG, sG, bG))
    return cudaErrorInvalidValue;
  const int cpt = int(ceil_div(p.R, kWKC));
  const int nchunks = p.T * cpt;
  if (int64_t(nchunks) * p.V * p.Nout > p.partial_cap) return cudaErrorInvalidValue;
  const dim3 grid(unsigned(ceil_div(p.V, kBM)), unsigned(nchunks));
  const int64_t n = int64_t(p.V) * p.Nout;
  {
    const double TR = double(p.T) * p.R;
    ProfScope prof(kProfGemmWgrad, s, 2.0 * TR * p.V + 2.0 * TR * p.Nout + 4.0 * nchunks * n,
                   2.0 * TR * p.V * p.Nout);
    if (p.Nout == 128) {
      static cudaError_t once = set_smem(k_tc_wgrad<128>, wg_smem_bytes(128));
      if (once != cudaSuccess) return once;
      k_tc_wgrad<128><<<grid, kWgThreads, wg_smem_bytes(128), s>>>(ma_in, ma_h, mg, p, cpt);
    } else {
      static cudaError_t once = set_smem(k_tc_wgrad<64>, wg_smem_bytes(64));
      if (once != cudaSuccess) return once;
      k_tc_wgrad<64><<<grid, kWgThreads, wg_smem_bytes(64), s>>>(ma_in, ma_h, mg, p, cpt);
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ProfScope prof(kProfReduce, s, 4.0 * double(n) * (nchunks + 1), double(n) * nchunks);
  k_tc_reduce<<<unsigned(std::min<int64_t>(ceil_div(n, 256), 1184)), 256, 0, s>>>(
      p.partial, nchunks, p.V, p.Nout, p.vseg, p.coff, p.C_in, p.out);
  return cudaGetLastError();
}

}  // namespace pgti
