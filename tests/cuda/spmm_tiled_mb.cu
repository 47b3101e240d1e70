// Microbenchmark (dev tool, not a test): the diffusion SpMM (K2) on a real synthetic sensor
// graph read from a CSR file: the global-gather kernel vs shared-memory staged window kernels
// (plan of pgti_graph_windows, rebuilt here on the host).
//   python tests/cuda/dump_csr.py pems_all_la /tmp/csr.bin
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tests/cuda/spmm_tiled_mb.cu -o /tmp/mb
//   /tmp/mb /tmp/csr.bin 4096
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstring>
#include <cmath>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("%s failed: %s\n", #x, cudaGetErrorString(e));                      \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

using bf16 = __nv_bfloat16;

__device__ __forceinline__ float2 unpack(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}
__device__ __forceinline__ void fma8(float2 *acc, float w, uint4 a) {
  const float2 ww = make_float2(w, w);
  acc[0] = __ffma2_rn(ww, unpack(a.x), acc[0]);
  acc[1] = __ffma2_rn(ww, unpack(a.y), acc[1]);
  acc[2] = __ffma2_rn(ww, unpack(a.z), acc[2]);
  acc[3] = __ffma2_rn(ww, unpack(a.w), acc[3]);
}
__device__ __forceinline__ uint4 pack(const float2 *acc) {
  uint4 o;
  __nv_bfloat162 h;
  h = __floats2bfloat162_rn(acc[0].x, acc[0].y), o.x = *reinterpret_cast<uint32_t *>(&h);
  h = __floats2bfloat162_rn(acc[1].x, acc[1].y), o.y = *reinterpret_cast<uint32_t *>(&h);
  h = __floats2bfloat162_rn(acc[2].x, acc[2].y), o.z = *reinterpret_cast<uint32_t *>(&h);
  h = __floats2bfloat162_rn(acc[3].x, acc[3].y), o.w = *reinterpret_cast<uint32_t *>(&h);
  return o;
}
__device__ __forceinline__ void cp_async16(void *smem, const void *g) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}

// global gather: thread per (node, 16-byte vector), 4 loads unrolled
__global__ void __launch_bounds__(256) kOld(const int *rp, const int *ci, const float *va,
                                            const bf16 *X, bf16 *Y, int N, int W) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, vecs = W / 8;
  if (tid >= N * vecs) return;
  const int n = tid / vecs, col0 = (tid % vecs) * 8;
  const bf16 *Xc = X + col0;
  float2 acc[4] = {};
  const int beg = __ldg(rp + n), end = __ldg(rp + n + 1);
  int e = beg;
  for (; e + 4 <= end; e += 4) {
    const int c0 = __ldg(ci + e), c1 = __ldg(ci + e + 1), c2 = __ldg(ci + e + 2), c3 = __ldg(ci + e + 3);
    const float w0 = __ldg(va + e), w1 = __ldg(va + e + 1), w2 = __ldg(va + e + 2), w3 = __ldg(va + e + 3);
    fma8(acc, w0, __ldg(reinterpret_cast<const uint4 *>(Xc + size_t(c0) * W)));
    fma8(acc, w1, __ldg(reinterpret_cast<const uint4 *>(Xc + size_t(c1) * W)));
    fma8(acc, w2, __ldg(reinterpret_cast<const uint4 *>(Xc + size_t(c2) * W)));
    fma8(acc, w3, __ldg(reinterpret_cast<const uint4 *>(Xc + size_t(c3) * W)));
  }
  for (; e < end; ++e) fma8(acc, __ldg(va + e), __ldg(reinterpret_cast<const uint4 *>(Xc + size_t(__ldg(ci + e)) * W)));
  *reinterpret_cast<uint4 *>(Y + size_t(n) * W + col0) = pack(acc);
}

// global gather with all of a row's loads in flight: CSR entries first (predicated), then up to
// U neighbour slices, then the FMAs in CSR order
template <int U>
__global__ void __launch_bounds__(256) kOldU(const int *rp, const int *ci, const float *va,
                                             const bf16 *X, bf16 *Y, int N, int W) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, vecs = W / 8;
  if (tid >= N * vecs) return;
  const int n = tid / vecs, col0 = (tid % vecs) * 8;
  const bf16 *Xc = X + col0;
  float2 acc[4] = {};
  const int beg = __ldg(rp + n), end = __ldg(rp + n + 1);
  for (int e0 = beg; e0 < end; e0 += U) {
    int c[U];
    float w[U];
    uint4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = e0 + u < end ? __ldg(ci + e0 + u) : 0;
      w[u] = e0 + u < end ? __ldg(va + e0 + u) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u < end) x[u] = __ldg(reinterpret_cast<const uint4 *>(Xc + size_t(c[u]) * W));
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u < end) fma8(acc, w[u], x[u]);
  }
  *reinterpret_cast<uint4 *>(Y + size_t(n) * W + col0) = pack(acc);
}

struct Plan {
  const int *rp;
  const float *va;
  const int *wptr, *wnodes;
  const uint16_t *lcol;
  int N, W, rows, nwin, maxu, maxe;
};

// staged, CPB chunks per CTA, NBUF stage buffers (NBUF = 2: chunk c+1 staged while c computes).
// Index loads (union node ids -> smem, each warp's rows' CSR -> registers) once per CTA.
template <int RPW, int CPB, int NBUF>
__global__ void __launch_bounds__(256) kWin(const Plan p, const bf16 *X, bf16 *Y) {
  extern __shared__ uint4 sm[];
  const int vecs = p.W / 8, nchunk = (vecs + 31) / 32, ngrp = (nchunk + CPB - 1) / CPB;
  const int grp = blockIdx.x % ngrp, win = blockIdx.x / ngrp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = win * p.rows;
  uint4 *stage = sm;
  int *s_nodes = reinterpret_cast<int *>(sm + NBUF * p.maxu * 32);
  const int ub = __ldg(p.wptr + win), nu = __ldg(p.wptr + win + 1) - ub;
  for (int i = threadIdx.x; i < nu; i += 256) s_nodes[i] = __ldg(p.wnodes + ub + i);
  int beg[RPW], cnt[RPW], cc[RPW];
  float cv[RPW];
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int r = warp + 8 * i, n = row0 + r;
    beg[i] = cnt[i] = cc[i] = 0, cv[i] = 0.f;
    if (r >= p.rows || n >= p.N) continue;
    beg[i] = __ldg(p.rp + n);
    cnt[i] = __ldg(p.rp + n + 1) - beg[i];
    if (lane < cnt[i]) cc[i] = __ldg(p.lcol + beg[i] + lane), cv[i] = __ldg(p.va + beg[i] + lane);
  }
  __syncthreads();
  const int c_lo = grp * CPB, c_hi = min(nchunk, c_lo + CPB);
  auto issue = [&](int c, int buf) {
    const int vec = c * 32 + lane;
    if (vec < vecs) {
      const bf16 *Xc = X + size_t(vec) * 8;
      uint4 *st = stage + buf * p.maxu * 32;
      for (int k = warp; k < nu; k += 8) cp_async16(st + k * 32 + lane, Xc + size_t(s_nodes[k]) * p.W);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll 1
  for (int b = 0; b < NBUF - 1 && c_lo + b < c_hi; ++b) issue(c_lo + b, b);
#pragma unroll 1
  for (int c = c_lo; c < c_hi; ++c) {
    const int buf = (c - c_lo) % NBUF;
    if (c + NBUF - 1 < c_hi) {
      issue(c + NBUF - 1, (c + NBUF - 1 - c_lo) % NBUF);
      asm volatile("cp.async.wait_group %0;" ::"n"(NBUF - 1) : "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const uint4 *st = stage + buf * p.maxu * 32;
    const int vec = c * 32 + lane;
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      const int r = warp + 8 * i, n = row0 + r;
      if (r >= p.rows || n >= p.N) continue;
      float2 acc[4] = {};
      const int n0 = min(cnt[i], 32);
      int u = 0;
      for (; u + 4 <= n0; u += 4) {
        const int c0 = __shfl_sync(~0u, cc[i], u), c1 = __shfl_sync(~0u, cc[i], u + 1),
                  c2 = __shfl_sync(~0u, cc[i], u + 2), c3 = __shfl_sync(~0u, cc[i], u + 3);
        const float w0 = __shfl_sync(~0u, cv[i], u), w1 = __shfl_sync(~0u, cv[i], u + 1),
                    w2 = __shfl_sync(~0u, cv[i], u + 2), w3 = __shfl_sync(~0u, cv[i], u + 3);
        fma8(acc, w0, st[c0 * 32 + lane]);
        fma8(acc, w1, st[c1 * 32 + lane]);
        fma8(acc, w2, st[c2 * 32 + lane]);
        fma8(acc, w3, st[c3 * 32 + lane]);
      }
      for (; u < n0; ++u) fma8(acc, __shfl_sync(~0u, cv[i], u), st[__shfl_sync(~0u, cc[i], u) * 32 + lane]);
      for (int e = beg[i] + 32; e < beg[i] + cnt[i]; ++e) fma8(acc, __ldg(p.va + e), st[__ldg(p.lcol + e) * 32 + lane]);
      if (vec < vecs) *reinterpret_cast<uint4 *>(Y + size_t(n) * p.W + size_t(vec) * 8) = pack(acc);
    }
    __syncthreads();  // buffer free before it is re-staged
  }
}

// v3: 2-D grid (x = 512-byte chunk, y = window: no integer division), the window's CSR staged in
// shared memory as (byte offset into the stage, value) pairs, read back with one broadcast LDS.64
// per entry; one chunk per CTA.
template <int RPW>
__global__ void __launch_bounds__(256) kWin3(const Plan p, const bf16 *X, bf16 *Y) {
  extern __shared__ uint4 sm[];
  const int vecs = p.W / 8;
  const int chunk = blockIdx.x, win = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = win * p.rows, nrows = min(p.rows, p.N - row0);
  const int ub = __ldg(p.wptr + win), nu = __ldg(p.wptr + win + 1) - ub;
  const int e0 = __ldg(p.rp + row0), e1 = __ldg(p.rp + row0 + nrows);
  uint4 *stage = sm;
  int *s_nodes = reinterpret_cast<int *>(sm + p.maxu * 32);
  int2 *s_ent = reinterpret_cast<int2 *>(s_nodes + p.maxu + (p.maxu & 1));
  int *s_rp = reinterpret_cast<int *>(s_ent + p.maxe);
  for (int i = threadIdx.x; i < nu; i += 256) s_nodes[i] = __ldg(p.wnodes + ub + i);
  for (int i = threadIdx.x; i < e1 - e0; i += 256)
    s_ent[i] = make_int2(int(__ldg(p.lcol + e0 + i)) * 512, __float_as_int(__ldg(p.va + e0 + i)));
  for (int i = threadIdx.x; i <= nrows; i += 256) s_rp[i] = __ldg(p.rp + row0 + i) - e0;
  __syncthreads();
  const int vec = chunk * 32 + lane;
  const bool act = vec < vecs;
  if (act) {
    const bf16 *Xc = X + size_t(vec) * 8;
    for (int k = warp; k < nu; k += 8) cp_async16(stage + k * 32 + lane, Xc + size_t(s_nodes[k]) * p.W);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const char *sb = reinterpret_cast<const char *>(stage) + lane * 16;
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int r = warp + 8 * i;
    if (r >= nrows) break;
    float2 acc[4] = {};
    const int b = s_rp[r], e = s_rp[r + 1];
    int q = b;
    for (; q + 2 <= e; q += 2) {
      const int2 a0 = s_ent[q], a1 = s_ent[q + 1];
      const uint4 x0 = *reinterpret_cast<const uint4 *>(sb + a0.x);
      const uint4 x1 = *reinterpret_cast<const uint4 *>(sb + a1.x);
      fma8(acc, __int_as_float(a0.y), x0);
      fma8(acc, __int_as_float(a1.y), x1);
    }
    if (q < e) {
      const int2 a0 = s_ent[q];
      fma8(acc, __int_as_float(a0.y), *reinterpret_cast<const uint4 *>(sb + a0.x));
    }
    if (act) *reinterpret_cast<uint4 *>(Y + size_t(row0 + r) * p.W + size_t(vec) * 8) = pack(acc);
  }
}

// v4: v3 with VPL 16-byte vectors per lane (chunk = VPL * 512 bytes) and NW warps per CTA
template <int RPW, int VPL, int NWARP>
__global__ void __launch_bounds__(NWARP * 32) kWin4(const Plan p, const bf16 *X, bf16 *Y) {
  extern __shared__ uint4 sm[];
  constexpr int CV = 32 * VPL;  // vectors per chunk
  const int vecs = p.W / 8;
  const int chunk = blockIdx.x, win = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = win * p.rows, nrows = min(p.rows, p.N - row0);
  const int ub = __ldg(p.wptr + win), nu = __ldg(p.wptr + win + 1) - ub;
  const int e0 = __ldg(p.rp + row0), e1 = __ldg(p.rp + row0 + nrows);
  uint4 *stage = sm;
  int *s_nodes = reinterpret_cast<int *>(sm + p.maxu * CV);
  int2 *s_ent = reinterpret_cast<int2 *>(s_nodes + p.maxu + (p.maxu & 1));
  int *s_rp = reinterpret_cast<int *>(s_ent + p.maxe);
  for (int i = threadIdx.x; i < nu; i += NWARP * 32) s_nodes[i] = __ldg(p.wnodes + ub + i);
  for (int i = threadIdx.x; i < e1 - e0; i += NWARP * 32)
    s_ent[i] = make_int2(int(__ldg(p.lcol + e0 + i)) * CV * 16, __float_as_int(__ldg(p.va + e0 + i)));
  for (int i = threadIdx.x; i <= nrows; i += NWARP * 32) s_rp[i] = __ldg(p.rp + row0 + i) - e0;
  __syncthreads();
  const int vbase = chunk * CV;
  for (int k = warp; k < nu; k += NWARP) {
    const bf16 *Xr = X + size_t(s_nodes[k]) * p.W;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int vec = vbase + v * 32 + lane;
      if (vec < vecs) cp_async16(stage + k * CV + v * 32 + lane, Xr + size_t(vec) * 8);
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const char *sb = reinterpret_cast<const char *>(stage) + lane * 16;
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int r = warp + NWARP * i;
    if (r >= nrows) break;
    float2 acc[VPL][4] = {};
    const int b = s_rp[r], e = s_rp[r + 1];
    for (int q = b; q < e; ++q) {
      const int2 a0 = s_ent[q];
      const float w = __int_as_float(a0.y);
#pragma unroll
      for (int v = 0; v < VPL; ++v) fma8(acc[v], w, *reinterpret_cast<const uint4 *>(sb + a0.x + v * 512));
    }
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int vec = vbase + v * 32 + lane;
      if (vec < vecs) *reinterpret_cast<uint4 *>(Y + size_t(row0 + r) * p.W + size_t(vec) * 8) = pack(acc[v]);
    }
  }
}

// global gather, persistent grid-stride: G CTAs per SM, each thread loops over (node, vector)
// work items (fewer CTAs to launch than one thread per item)
__global__ void __launch_bounds__(256) kOldGS(const int *rp, const int *ci, const float *va,
                                              const bf16 *X, bf16 *Y, int N, int W) {
  const int vecs = W / 8;
  const int total = N * vecs;
  for (int tid = blockIdx.x * blockDim.x + threadIdx.x; tid < total; tid += gridDim.x * blockDim.x) {
    const int n = tid / vecs, col0 = (tid % vecs) * 8;
    const bf16 *Xc = X + col0;
    float2 acc[4] = {};
    const int beg = __ldg(rp + n), end = __ldg(rp + n + 1);
    int e = beg;
    for (; e + 4 <= end; e += 4) {
      const int c0 = __ldg(ci + e), c1 = __ldg(ci + e + 1), c2 = __ldg(ci + e + 2), c3 = __ldg(ci + e + 3);
      const float w0 = __ldg(va + e), w1 = __ldg(va + e + 1), w2 = __ldg(va + e + 2), w3 = __ldg(va + e + 3);
      fma8(acc, w0, __ldg(reinterpret_cast<const uint4 *>(Xc + size_t(c0) * W)));
      fma8(acc, w1, __ldg(reinterpret_cast<const uint4 *>(Xc + size_t(c1) * W)));
      fma8(acc, w2, __ldg(reinterpret_cast<const uint4 *>(Xc + size_t(c2) * W)));
      fma8(acc, w3, __ldg(reinterpret_cast<const uint4 *>(Xc + size_t(c3) * W)));
    }
    for (; e < end; ++e) fma8(acc, __ldg(va + e), __ldg(reinterpret_cast<const uint4 *>(Xc + size_t(__ldg(ci + e)) * W)));
    *reinterpret_cast<uint4 *>(Y + size_t(n) * W + col0) = pack(acc);
  }
}

// v3 with bf16 weights and mixed-precision FMA (fma.rn.f32.bf16 -> FHFMA.BF16): each bf16 of the
// neighbour slice is multiplied in place (no unpack), fp32 accumulation
__device__ __forceinline__ float fhfma_lo(uint32_t x, uint32_t w2, float acc) {
  float r;
  asm("fma.rn.f32.bf16 %0, %1, %2, %3;" : "=f"(r) : "h"((unsigned short)(x & 0xffff)),
      "h"((unsigned short)(w2 & 0xffff)), "f"(acc));
  return r;
}
__device__ __forceinline__ float fhfma_hi(uint32_t x, uint32_t w2, float acc) {
  float r;
  asm("fma.rn.f32.bf16 %0, %1, %2, %3;" : "=f"(r) : "h"((unsigned short)(x >> 16)),
      "h"((unsigned short)(w2 & 0xffff)), "f"(acc));
  return r;
}
template <int RPW>
__global__ void __launch_bounds__(256) kWin3h(const Plan p, const bf16 *X, bf16 *Y) {
  extern __shared__ uint4 sm[];
  const int vecs = p.W / 8;
  const int chunk = blockIdx.x, win = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = win * p.rows, nrows = min(p.rows, p.N - row0);
  const int ub = __ldg(p.wptr + win), nu = __ldg(p.wptr + win + 1) - ub;
  const int e0 = __ldg(p.rp + row0), e1 = __ldg(p.rp + row0 + nrows);
  uint4 *stage = sm;
  int *s_nodes = reinterpret_cast<int *>(sm + p.maxu * 32);
  int2 *s_ent = reinterpret_cast<int2 *>(s_nodes + p.maxu + (p.maxu & 1));
  int *s_rp = reinterpret_cast<int *>(s_ent + p.maxe);
  for (int i = threadIdx.x; i < nu; i += 256) s_nodes[i] = __ldg(p.wnodes + ub + i);
  for (int i = threadIdx.x; i < e1 - e0; i += 256) {
    const __nv_bfloat16 wb = __float2bfloat16_rn(__ldg(p.va + e0 + i));
    s_ent[i] = make_int2(int(__ldg(p.lcol + e0 + i)) * 512, int(*reinterpret_cast<const unsigned short *>(&wb)));
  }
  for (int i = threadIdx.x; i <= nrows; i += 256) s_rp[i] = __ldg(p.rp + row0 + i) - e0;
  __syncthreads();
  const int vec = chunk * 32 + lane;
  const bool act = vec < vecs;
  if (act) {
    const bf16 *Xc = X + size_t(vec) * 8;
    for (int k = warp; k < nu; k += 8) cp_async16(stage + k * 32 + lane, Xc + size_t(s_nodes[k]) * p.W);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const char *sb = reinterpret_cast<const char *>(stage) + lane * 16;
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int r = warp + 8 * i;
    if (r >= nrows) break;
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const int b = s_rp[r], e = s_rp[r + 1];
    for (int q = b; q < e; ++q) {
      const int2 en = s_ent[q];
      const uint4 x = *reinterpret_cast<const uint4 *>(sb + en.x);
      const uint32_t w2 = uint32_t(en.y);
      a[0] = fhfma_lo(x.x, w2, a[0]), a[1] = fhfma_hi(x.x, w2, a[1]);
      a[2] = fhfma_lo(x.y, w2, a[2]), a[3] = fhfma_hi(x.y, w2, a[3]);
      a[4] = fhfma_lo(x.z, w2, a[4]), a[5] = fhfma_hi(x.z, w2, a[5]);
      a[6] = fhfma_lo(x.w, w2, a[6]), a[7] = fhfma_hi(x.w, w2, a[7]);
    }
    float2 acc[4] = {make_float2(a[0], a[1]), make_float2(a[2], a[3]), make_float2(a[4], a[5]),
                     make_float2(a[6], a[7])};
    if (act) *reinterpret_cast<uint4 *>(Y + size_t(row0 + r) * p.W + size_t(vec) * 8) = pack(acc);
  }
}

// v5: v3 with CPB column chunks per CTA processed one after the other through one stage buffer
// (the window's index prologue amortised over CPB chunks)
template <int RPW, int CPB>
__global__ void __launch_bounds__(256) kWin5(const Plan p, const bf16 *X, bf16 *Y) {
  extern __shared__ uint4 sm[];
  const int vecs = p.W / 8, nchunk = (vecs + 31) / 32;
  const int win = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = win * p.rows, nrows = min(p.rows, p.N - row0);
  const int ub = __ldg(p.wptr + win), nu = __ldg(p.wptr + win + 1) - ub;
  const int e0 = __ldg(p.rp + row0), e1 = __ldg(p.rp + row0 + nrows);
  uint4 *stage = sm;
  int *s_nodes = reinterpret_cast<int *>(sm + p.maxu * 32);
  int2 *s_ent = reinterpret_cast<int2 *>(s_nodes + p.maxu + (p.maxu & 1));
  int *s_rp = reinterpret_cast<int *>(s_ent + p.maxe);
  for (int i = threadIdx.x; i < nu; i += 256) s_nodes[i] = __ldg(p.wnodes + ub + i);
  for (int i = threadIdx.x; i < e1 - e0; i += 256)
    s_ent[i] = make_int2(int(__ldg(p.lcol + e0 + i)) * 512, __float_as_int(__ldg(p.va + e0 + i)));
  for (int i = threadIdx.x; i <= nrows; i += 256) s_rp[i] = __ldg(p.rp + row0 + i) - e0;
  __syncthreads();
  const char *sb = reinterpret_cast<const char *>(stage) + lane * 16;
  for (int cc = 0; cc < CPB; ++cc) {
    const int chunk = blockIdx.x * CPB + cc;
    if (chunk >= nchunk) break;
    const int vec = chunk * 32 + lane;
    const bool act = vec < vecs;
    if (cc) __syncthreads();
    if (act) {
      const bf16 *Xc = X + size_t(vec) * 8;
      for (int k = warp; k < nu; k += 8) cp_async16(stage + k * 32 + lane, Xc + size_t(s_nodes[k]) * p.W);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
      const int r = warp + 8 * i;
      if (r >= nrows) break;
      float2 acc[4] = {};
      const int b = s_rp[r], e = s_rp[r + 1];
      int q = b;
      for (; q + 2 <= e; q += 2) {
        const int2 a0 = s_ent[q], a1 = s_ent[q + 1];
        const uint4 x0 = *reinterpret_cast<const uint4 *>(sb + a0.x);
        const uint4 x1 = *reinterpret_cast<const uint4 *>(sb + a1.x);
        fma8(acc, __int_as_float(a0.y), x0);
        fma8(acc, __int_as_float(a1.y), x1);
      }
      if (q < e) {
        const int2 a0 = s_ent[q];
        fma8(acc, __int_as_float(a0.y), *reinterpret_cast<const uint4 *>(sb + a0.x));
      }
      if (act) *reinterpret_cast<uint4 *>(Y + size_t(row0 + r) * p.W + size_t(vec) * 8) = pack(acc);
    }
  }
}

__global__ void kCopy(const uint4 *X, uint4 *Y, size_t n) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i < n) Y[i] = X[i];
}

int main(int argc, char **argv) {
  if (argc < 2) return 1;
  const int W = argc > 2 ? atoi(argv[2]) : 4096;
  FILE *f = fopen(argv[1], "rb");
  int N, nnz;
  if (fread(&N, 4, 1, f) != 1 || fread(&nnz, 4, 1, f) != 1) return 1;
  std::vector<int> rp(N + 1), ci(nnz);
  std::vector<float> va(nnz);
  if (fread(rp.data(), 4, N + 1, f) != size_t(N + 1) || fread(ci.data(), 4, nnz, f) != size_t(nnz) ||
      fread(va.data(), 4, nnz, f) != size_t(nnz))
    return 1;
  fclose(f);
  printf("N=%d nnz=%d W=%d (%.1f nnz/row)  X=%.1f MB\n", N, nnz, W, double(nnz) / N, N * double(W) * 2 / 1e6);
  int *d_rp, *d_ci;
  float *d_va;
  bf16 *X, *Y, *Y0;
  CK(cudaMalloc(&d_rp, rp.size() * 4));
  CK(cudaMalloc(&d_ci, ci.size() * 4));
  CK(cudaMalloc(&d_va, va.size() * 4));
  const size_t nel = size_t(N) * W;
  CK(cudaMalloc(&X, nel * 2));
  CK(cudaMalloc(&Y, nel * 2));
  CK(cudaMalloc(&Y0, nel * 2));
  CK(cudaMemcpy(d_rp, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_ci, ci.data(), ci.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_va, va.data(), va.size() * 4, cudaMemcpyHostToDevice));
  {
    std::vector<bf16> h(nel);
    for (size_t i = 0; i < nel; ++i) h[i] = __float2bfloat16(float((i * 2654435761u) % 1000) / 500.f - 1.f);
    CK(cudaMemcpy(X, h.data(), nel * 2, cudaMemcpyHostToDevice));
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a), cudaEventCreate(&b);
  const double bytes = nel * 2.0 * 2 + nnz * 8.0;
  auto time = [&](const char *name, auto launch) {
    for (int i = 0; i < 10; ++i) launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int i = 0; i < 100; ++i) launch();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1000 / 100;
    printf("%-34s %8.2f us  %7.0f GB/s (algorithmic)\n", name, us, bytes / us / 1e3);
  };
  auto check = [&](const char *name) {
    std::vector<uint16_t> h0(nel), h1(nel);
    CK(cudaMemcpy(h0.data(), Y0, nel * 2, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h1.data(), Y, nel * 2, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (size_t i = 0; i < nel; ++i) bad += h0[i] != h1[i];
    if (bad) printf("  %s: %zu MISMATCHES\n", name, bad);
  };
  const int vecs = W / 8;
  time("copy", [&] {
    kCopy<<<unsigned((nel / 8 + 255) / 256), 256>>>((const uint4 *)X, (uint4 *)Y, nel / 8);
  });
  time("global gather (old)", [&] { kOld<<<unsigned((N * vecs + 255) / 256), 256>>>(d_rp, d_ci, d_va, X, Y0, N, W); });
  for (int g : {1, 2, 4, 8}) {
    char nm[48];
    snprintf(nm, 48, "gather grid-stride %d CTA/SM", g);
    time(nm, [&] { kOldGS<<<148 * g, 256>>>(d_rp, d_ci, d_va, X, Y, N, W); });
    check(nm);
  }
  time("global gather U=8", [&] { kOldU<8><<<unsigned((N * vecs + 255) / 256), 256>>>(d_rp, d_ci, d_va, X, Y, N, W); });
  check("U=8");
  time("global gather U=12", [&] { kOldU<12><<<unsigned((N * vecs + 255) / 256), 256>>>(d_rp, d_ci, d_va, X, Y, N, W); });
  check("U=12");
  time("global gather U=16 128thr", [&] { kOldU<16><<<unsigned((N * vecs + 127) / 128), 128>>>(d_rp, d_ci, d_va, X, Y, N, W); });
  check("U=16");
  const int nchunk = (vecs + 31) / 32;
  for (int rows : {16, 32, 64}) {
    const int nwin = (N + rows - 1) / rows;
    std::vector<int> wptr(nwin + 1), wn;
    std::vector<uint16_t> lc(nnz);
    int maxu = 0;
    for (int w = 0; w < nwin; ++w) {
      const int r0 = w * rows, r1 = std::min(N, r0 + rows);
      std::vector<int> u(ci.begin() + rp[r0], ci.begin() + rp[r1]);
      std::sort(u.begin(), u.end());
      u.erase(std::unique(u.begin(), u.end()), u.end());
      for (int e = rp[r0]; e < rp[r1]; ++e) lc[e] = uint16_t(std::lower_bound(u.begin(), u.end(), ci[e]) - u.begin());
      wptr[w] = int(wn.size());
      wn.insert(wn.end(), u.begin(), u.end());
      maxu = std::max(maxu, int(u.size()));
    }
    wptr[nwin] = int(wn.size());
    int *d_wp, *d_wn;
    uint16_t *d_lc;
    CK(cudaMalloc(&d_wp, wptr.size() * 4));
    CK(cudaMalloc(&d_wn, wn.size() * 4));
    CK(cudaMalloc(&d_lc, lc.size() * 2));
    CK(cudaMemcpy(d_wp, wptr.data(), wptr.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_wn, wn.data(), wn.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_lc, lc.data(), lc.size() * 2, cudaMemcpyHostToDevice));
    int maxe = 0;
    for (int w = 0; w < nwin; ++w) maxe = std::max(maxe, rp[std::min(N, (w + 1) * rows)] - rp[w * rows]);
    Plan p{d_rp, d_va, d_wp, d_wn, d_lc, N, W, rows, nwin, maxu, maxe};
    printf("rows=%d maxu=%d union/rows=%.2f\n", rows, maxu, double(wn.size()) / N);
#define RUN(RPW, CPB, NBUF)                                                                      \
  if ((rows + 7) / 8 == RPW) {                                                                   \
    const int smem = NBUF * maxu * 512 + maxu * 4;                                               \
    CK(cudaFuncSetAttribute(kWin<RPW, CPB, NBUF>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
    const int grid = nwin * ((nchunk + CPB - 1) / CPB);                                          \
    char nm[64];                                                                                 \
    snprintf(nm, 64, "  win RPW=%d CPB=%d NBUF=%d (%d CTAs)", RPW, CPB, NBUF, grid);             \
    time(nm, [&] { kWin<RPW, CPB, NBUF><<<grid, 256, smem>>>(p, X, Y); });                       \
    check(nm);                                                                                   \
  }
    RUN(2, 1, 1) RUN(4, 1, 1) RUN(8, 1, 1)
#define RUN3(RPW)                                                                                \
  if ((rows + 7) / 8 == RPW) {                                                                   \
    const int smem = maxu * 512 + (maxu + 1) * 4 + maxe * 8 + (rows + 1) * 4 + 16;               \
    CK(cudaFuncSetAttribute(kWin3<RPW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));    \
    char nm[64];                                                                                 \
    snprintf(nm, 64, "  v3 RPW=%d (%d CTAs)", RPW, nwin * nchunk);                               \
    time(nm, [&] { kWin3<RPW><<<dim3(nchunk, nwin), 256, smem>>>(p, X, Y); });                   \
    check(nm);                                                                                   \
  }
    RUN3(2) RUN3(4) RUN3(8)
#define RUN3H(RPW)                                                                               \
  if ((rows + 7) / 8 == RPW) {                                                                   \
    const int smem = maxu * 512 + (maxu + 1) * 4 + maxe * 8 + (rows + 1) * 4 + 16;               \
    CK(cudaFuncSetAttribute(kWin3h<RPW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));   \
    char nm[64];                                                                                 \
    snprintf(nm, 64, "  v3 bf16-w FHFMA RPW=%d", RPW);                                           \
    time(nm, [&] { kWin3h<RPW><<<dim3(nchunk, nwin), 256, smem>>>(p, X, Y); });                  \
    { std::vector<uint16_t> h0(nel), h1(nel);                                                    \
      CK(cudaMemcpy(h0.data(), Y0, nel * 2, cudaMemcpyDeviceToHost));                            \
      CK(cudaMemcpy(h1.data(), Y, nel * 2, cudaMemcpyDeviceToHost));                             \
      double mx = 0; for (size_t i = 0; i < nel; ++i) { uint32_t u0 = uint32_t(h0[i]) << 16,    \
        u1 = uint32_t(h1[i]) << 16; float f0, f1; memcpy(&f0, &u0, 4); memcpy(&f1, &u1, 4);      \
        mx = std::max(mx, double(fabsf(f0 - f1))); }                                             \
      printf("    max |diff| vs fp32-weight result: %.3g\n", mx); }                               \
  }
    RUN3H(2) RUN3H(4)
#define RUN5(RPW, CPB)                                                                           \
  if ((rows + 7) / 8 == RPW) {                                                                   \
    const int smem = maxu * 512 + (maxu + 1) * 4 + maxe * 8 + (rows + 1) * 4 + 16;               \
    CK(cudaFuncSetAttribute(kWin5<RPW, CPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
    char nm[64];                                                                                 \
    snprintf(nm, 64, "  v5 RPW=%d CPB=%d (%d CTAs)", RPW, CPB, nwin * ((nchunk + CPB - 1) / CPB)); \
    time(nm, [&] { kWin5<RPW, CPB><<<dim3((nchunk + CPB - 1) / CPB, nwin), 256, smem>>>(p, X, Y); }); \
    check(nm);                                                                                   \
  }
    RUN5(2, 1) RUN5(2, 2) RUN5(2, 4) RUN5(4, 1) RUN5(4, 2) RUN5(4, 4)
#define RUN4(RPW, VPL, NWARP)                                                                    \
  if ((rows + NWARP - 1) / NWARP == RPW) {                                                       \
    const int smem = maxu * 512 * VPL + (maxu + 1) * 4 + maxe * 8 + (rows + 1) * 4 + 16;         \
    CK(cudaFuncSetAttribute(kWin4<RPW, VPL, NWARP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
    char nm[64];                                                                                 \
    const int nch = (vecs + 32 * VPL - 1) / (32 * VPL);                                          \
    snprintf(nm, 64, "  v4 RPW=%d VPL=%d NW=%d (%d CTAs)", RPW, VPL, NWARP, nwin * nch);         \
    time(nm, [&] { kWin4<RPW, VPL, NWARP><<<dim3(nch, nwin), NWARP * 32, smem>>>(p, X, Y); });  \
    check(nm);                                                                                   \
  }
    RUN4(2, 1, 8) RUN4(2, 2, 8) RUN4(1, 1, 16) RUN4(1, 2, 16)
    RUN4(4, 1, 8) RUN4(4, 2, 8) RUN4(2, 1, 16) RUN4(2, 2, 16)
    RUN4(8, 1, 8) RUN4(4, 1, 16) RUN4(4, 2, 16)
  }
  return 0;
}
