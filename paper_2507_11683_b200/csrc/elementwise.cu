// Small fused elementwise kernels of the step: x re-layout, MAE loss (K5), GRU backward.
#include <cuda_bf16.h>

#include "kernels.cuh"
#include "tc_ptx.cuh"
#include "profile.cuh"

namespace pgti {
namespace {

constexpr int kT = 256;

inline unsigned grid_for(int64_t n, int cap = 148 * 16) {
  return unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kT), cap)));
}

// x[b][t][ld] (gathered batch, sample-major) -> X0[t][n][b][f] (node-major rows = n*B + b,
// the dense-operand layout of the diffusion SpMM and the row order of the gate GEMMs).
// Row t of sample b's slice (nullptr if the window is not held: caller reads zeros).
__device__ __forceinline__ const float *win_row(const WindowSrc &w, int b, int t, int T,
                                                int64_t ld) {
  if (!w.idx) return w.base + (int64_t(b) * T + t) * ld;
  const int64_t s = int64_t(w.idx[b]) - w.row0;
  if (s < 0 || s + w.span > w.nrows) return nullptr;
  return w.base + (s + w.toff + t) * ld;
}

__global__ void k_x_prep(const __grid_constant__ WindowSrc xs, int B, int T_in, int64_t ld,
                         int N, int F, float *__restrict__ X0, unsigned *__restrict__ err) {
  const int64_t total = int64_t(T_in) * N * B * F;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    int64_t q = i;
    const int f = int(q % F);
    q /= F;
    const int b = int(q % B);
    q /= B;
    const int n = int(q % N);
    const int t = int(q / N);
    const float *row = win_row(xs, b, t, T_in, ld);
    if (!row && n == 0 && f == 0 && t == 0) atomicOr(err, kDevErrRange);
    X0[i] = row ? row[int64_t(n) * F + f] : 0.f;
  }
}

__global__ void k_dec_input(const __grid_constant__ WindowSrc ys, int tt, int B, int64_t ld,
                            int N, int F, int F_out, int T_out, float *__restrict__ out) {
  const int64_t total = int64_t(N) * B * F_out;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int o = int(i % F_out);
    const int64_t row = i / F_out;
    const int n = int(row / B), b = int(row % B);
    const float *yr = win_row(ys, b, tt, T_out, ld);
    out[i] = yr ? yr[int64_t(n) * F + o] : 0.f;
  }
}

// loss = mean |yhat - y[..., :F_out]|; dyhat = sign(resid) / count (0 at ties).
// yhat/dyhat [T_out][N*B][F_out] (row n*B + b); y [B][T_out][ld].
__global__ void k_loss_partial(const float *__restrict__ yhat, const __grid_constant__ WindowSrc ys,
                               int T_out, int N, int B, int F, int F_out, int64_t ld,
                               float *__restrict__ dyhat, double *__restrict__ partials) {
  griddep_launch_dependents();
  griddep_wait();
  const int64_t R = int64_t(N) * B, total = int64_t(T_out) * R * F_out;
  const float inv = float(1.0 / double(total));
  double acc = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int o = int(i % F_out);
    const int64_t rt = i / F_out;
    const int64_t row = rt % R;
    const int tt = int(rt / R);
    const int n = int(row / B), b = int(row % B);
    const float *yr = win_row(ys, b, tt, T_out, ld);
    const float yv = yr ? yr[int64_t(n) * F + o] : 0.f;
    const float r = yhat[i] - yv;
    dyhat[i] = r > 0.f ? inv : (r < 0.f ? -inv : 0.f);
    acc += double(fabsf(r));
  }
  __shared__ double red[kT / 32];
  for (int q = 16; q > 0; q >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, q);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kT / 32; ++w) s += red[w];
    partials[blockIdx.x] = s;
  }
}

__global__ void k_loss_final(const double *__restrict__ partials, int n, int64_t count,
                             float *__restrict__ loss, unsigned *__restrict__ err) {
  griddep_launch_dependents();
  griddep_wait();
  if (threadIdx.x != 0) return;
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += partials[i];
  const float l = float(s / double(count));
  *loss = l;
  if (!isfinite(l)) atomicOr(err, kDevErrNonfinite);
}

// Candidate / update backward:  H' = u H + (1-u) c,  c = tanh(pre)
//   dH' = dHcur (+ dyhat W_out^T);  dU = dH' (H - c);  dCpre = dH' (1-u)(1-c^2);  dHprev = dH' u
// (dCb: optional bf16 copy of dCpre -- the tensor-core dgrad / wgrad operand)
__global__ void k_cand_bwd(int64_t RH, int H, const float *__restrict__ dHcur,
                           const float *__restrict__ dHcur2,
                           const float *__restrict__ dy, const float *__restrict__ Wout, int F_out,
                           const float *__restrict__ u, const float *__restrict__ c,
                           const float *__restrict__ Hprev, float *__restrict__ dU,
                           float *__restrict__ dC, float *__restrict__ dHprev,
                           __nv_bfloat16 *__restrict__ dCb) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < RH;
       i += int64_t(gridDim.x) * blockDim.x) {
    float dh = dHcur ? dHcur[i] : 0.f;
    if (dHcur2) dh += dHcur2[i];
    if (dy) {
      const int64_t row = i / H;
      const int j = int(i - row * H);
      for (int o = 0; o < F_out; ++o) dh = fmaf(dy[row * F_out + o], Wout[j * F_out + o], dh);
    }
    const float uu = u[i], cc = c[i], hp = Hprev ? Hprev[i] : 0.f;
    dU[i] = dh * (hp - cc);
    const float dc = dh * (1.0f - uu) * (1.0f - cc * cc);
    dC[i] = dc;
    if (dCb) dCb[i] = __float2bfloat16_rn(dc);
    if (dHprev) dHprev[i] = dh * uu;
  }
}

// Tensor-core path candidate backward: as k_cand_bwd, plus the update-gate half of the gate
// gradient dG_u = dU u (1-u) (dU never leaves registers) and, when H_{t-1} = 0, dG_r = 0; the
// reset half dG_r is finished by the candidate dgrad GEMM's epilogue (TcFwd::fuse_tile).
// Thread = 4 consecutive hidden units of one row (16-byte loads / stores, 8-byte bf16 stores).
// The fp32 copies dC / dG are optional (the tensor-core path keeps only the bf16 ones).
__device__ __forceinline__ void st4bf(__nv_bfloat16 *p, float a, float b, float c, float d) {
  __nv_bfloat162 x = __floats2bfloat162_rn(a, b), y = __floats2bfloat162_rn(c, d);
  uint2 v;
  v.x = *reinterpret_cast<uint32_t *>(&x);
  v.y = *reinterpret_cast<uint32_t *>(&y);
  *reinterpret_cast<uint2 *>(p) = v;
}

__global__ void k_cand_bwd_tc(int64_t RH, int H, const float *__restrict__ dHa,
                              const float *__restrict__ dHb, const float *__restrict__ dy,
                              const float *__restrict__ Wout, int F_out,
                              const float *__restrict__ u, const __nv_bfloat16 *__restrict__ c,
                              const float *__restrict__ Hprev, float *__restrict__ dC,
                              __nv_bfloat16 *__restrict__ dCb, float *__restrict__ dHprev,
                              float *__restrict__ dG, __nv_bfloat16 *__restrict__ dGb) {
  griddep_launch_dependents();
  griddep_wait();
  const int64_t n4 = RH / 4;
  auto ld = [](const float *p, int64_t q) { return reinterpret_cast<const float4 *>(p)[q]; };
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n4;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = q * 4, row = i / H;
    const int j = int(i - row * H);
    float4 dh = dHa ? ld(dHa, q) : make_float4(0.f, 0.f, 0.f, 0.f);
    if (dHb) {
      const float4 b = ld(dHb, q);
      dh.x += b.x, dh.y += b.y, dh.z += b.z, dh.w += b.w;
    }
    if (dy)
      for (int o = 0; o < F_out; ++o) {
        const float e = dy[row * F_out + o];
        dh.x = fmaf(e, Wout[(j + 0) * F_out + o], dh.x);
        dh.y = fmaf(e, Wout[(j + 1) * F_out + o], dh.y);
        dh.z = fmaf(e, Wout[(j + 2) * F_out + o], dh.z);
        dh.w = fmaf(e, Wout[(j + 3) * F_out + o], dh.w);
      }
    const float4 uu = ld(u, q);
    float4 cc;
    {
      const uint2 cw = reinterpret_cast<const uint2 *>(c)[q];
      const float2 c0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&cw.x));
      const float2 c1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&cw.y));
      cc = make_float4(c0.x, c0.y, c1.x, c1.y);
    }
    const float4 hp = Hprev ? ld(Hprev, q) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 dc = make_float4(dh.x * (1.0f - uu.x) * (1.0f - cc.x * cc.x),
                                  dh.y * (1.0f - uu.y) * (1.0f - cc.y * cc.y),
                                  dh.z * (1.0f - uu.z) * (1.0f - cc.z * cc.z),
                                  dh.w * (1.0f - uu.w) * (1.0f - cc.w * cc.w));
    if (dC) reinterpret_cast<float4 *>(dC)[q] = dc;
    st4bf(dCb + i, dc.x, dc.y, dc.z, dc.w);
    if (dHprev)
      reinterpret_cast<float4 *>(dHprev)[q] =
          make_float4(dh.x * uu.x, dh.y * uu.y, dh.z * uu.z, dh.w * uu.w);
    const float4 gu = make_float4(dh.x * (hp.x - cc.x) * uu.x * (1.0f - uu.x),
                                  dh.y * (hp.y - cc.y) * uu.y * (1.0f - uu.y),
                                  dh.z * (hp.z - cc.z) * uu.z * (1.0f - uu.z),
                                  dh.w * (hp.w - cc.w) * uu.w * (1.0f - uu.w));
    const int64_t gi = row * 2 * H + H + j;
    if (dG) *reinterpret_cast<float4 *>(dG + gi) = gu;
    st4bf(dGb + gi, gu.x, gu.y, gu.z, gu.w);
    if (!Hprev) {
      if (dG) *reinterpret_cast<float4 *>(dG + gi - H) = make_float4(0.f, 0.f, 0.f, 0.f);
      st4bf(dGb + gi - H, 0.f, 0.f, 0.f, 0.f);
    }
  }
}

// Gate backward: rH = r*H;  dr = d(rH) H;  dHprev += d(rH) r;
//   dG[:, :H] = dr r (1-r),  dG[:, H:] = dU u (1-u)      (dGb: optional bf16 copy)
__global__ void k_gate_bwd(int64_t RH, int H, const float *__restrict__ drH,
                           const float *__restrict__ Hprev, const float *__restrict__ r,
                           const float *__restrict__ u, const float *__restrict__ dU,
                           float *__restrict__ dHprev, float *__restrict__ dG,
                           __nv_bfloat16 *__restrict__ dGb) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < RH;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = i / H;
    const int j = int(i - row * H);
    const float rr = r[i], uu = u[i];
    float dr = 0.f;
    if (drH) {
      const float d = drH[i];
      dr = Hprev ? d * Hprev[i] : 0.f;
      if (dHprev) dHprev[i] += d * rr;
    }
    const float g0 = dr * rr * (1.0f - rr), g1 = dU[i] * uu * (1.0f - uu);
    dG[row * 2 * H + j] = g0;
    dG[row * 2 * H + H + j] = g1;
    if (dGb) {
      dGb[row * 2 * H + j] = __float2bfloat16_rn(g0);
      dGb[row * 2 * H + H + j] = __float2bfloat16_rn(g1);
    }
  }
}

struct WeightParams {
  WeightJob job[8];
  int njobs;
};

// Per job: Wf[kb][j][c] (kb over the k-blocks of the tensor-core forward GEMM) and
// Wd[v][j] (rows of the tensor-core dgrad); grid-stride over Wf then Wd elements.
__global__ void k_convert_weights(const __grid_constant__ WeightParams p) {
  for (int q = 0; q < p.njobs; ++q) {
    const WeightJob &w = p.job[q];
    const int nkb = w.layer0 ? w.M + 1 : 2 * w.M;
    const int64_t nf = int64_t(nkb) * w.Nout * 64;
    __nv_bfloat16 *wf = static_cast<__nv_bfloat16 *>(w.Wf);
    __nv_bfloat16 *wd = static_cast<__nv_bfloat16 *>(w.Wd);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nf;
         i += int64_t(gridDim.x) * blockDim.x) {
      const int c = int(i % 64);
      const int j = int((i / 64) % w.Nout);
      const int kb = int(i / (64 * w.Nout));
      if (w.layer0 && kb == w.M) {  // the x k-block: column c = m*Fin + f
        const int m = c / w.Fin, f = c - m * w.Fin;
        wf[i] = c < w.M * w.Fin ? __float2bfloat16_rn(w.W[int64_t(m * w.C_in + f) * w.Nout + j])
                                : __float2bfloat16_rn(0.f);
        continue;
      }
      const int row = w.layer0 ? kb * w.C_in + w.Fin + c : (kb / 2) * w.C_in + (kb % 2) * 64 + c;
      wf[i] = __float2bfloat16_rn(w.W[int64_t(row) * w.Nout + j]);
    }
    const int vseg = w.layer0 ? 64 : w.C_in, coff = w.layer0 ? w.Fin : 0;
    const int64_t nd = int64_t(w.M) * vseg * w.Nout;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nd;
         i += int64_t(gridDim.x) * blockDim.x) {
      const int j = int(i % w.Nout);
      const int v = int(i / w.Nout);
      const int row = (v / vseg) * w.C_in + coff + v % vseg;
      wd[i] = __float2bfloat16_rn(w.W[int64_t(row) * w.Nout + j]);
    }
  }
}

}  // namespace

namespace {
// grid.y = time step; thread = 8 columns (16 bytes) of one row of Xb (32-bit index math)
__global__ void k_xpack(const float *__restrict__ Dx, int64_t x_mstride, int R, int F, int M,
                        __nv_bfloat16 *__restrict__ Xb) {
  // 8 lanes per row r of step t, lane o packing channels 8o..8o+7 (the M F diffused channels, then
  // a constant 1 at channel M F: its forward weight row is zero, its weight-gradient row is the
  // bias gradient sum_t,r dG; zero beyond): each row's 128 bytes are one coalesced store
  griddep_launch_dependents();
  griddep_wait();
  const int t = blockIdx.y, mf = M * F, o = threadIdx.x & 7;
  const float *src = Dx + int64_t(t) * R * F;
  const int m0 = (o * 8) / F, f0 = o * 8 - m0 * F;  // channel 8o = m0 F + f0
  const int rows_per_iter = gridDim.x * (blockDim.x >> 3);
  for (int r = blockIdx.x * (blockDim.x >> 3) + (threadIdx.x >> 3); r < R; r += rows_per_iter) {
    uint4 w = make_uint4(0u, 0u, 0u, 0u);
    if (o * 8 <= mf) {
      float v[8];
      int m = m0, f = f0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int c = o * 8 + k;
        v[k] = c < mf ? __ldg(src + m * x_mstride + int64_t(r) * F + f) : c == mf ? 1.f : 0.f;
        if (++f == F) f = 0, ++m;
      }
      w = tc::pack8_bf16(v);
    }
    reinterpret_cast<uint4 *>(Xb + (int64_t(t) * R + r) * 64)[o] = w;
  }
}
}  // namespace

cudaError_t launch_xpack(const float *Dx, int64_t x_mstride, int T, int64_t R, int F, int M,
                         __nv_bfloat16 *Xb, cudaStream_t s) {
  if (M * F > 64 || R * 8 >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
  ProfScope prof(kProfElementwise, s, double(T) * R * (4.0 * M * F + 128.0), 0.0);
  const dim3 grid(unsigned(std::min<int64_t>(ceil_div(R * 8, kT), 4 * 148)), unsigned(T));
  return pdl_launch(k_xpack, grid, dim3(kT), 0, s, Dx, x_mstride, int(R), F, M, Xb);
}

cudaError_t launch_x_prep(const WindowSrc &xs, int B, int T_in, int64_t ld, int N, int F,
                          float *X0, unsigned *err, cudaStream_t s) {
  const int64_t n = int64_t(T_in) * N * B * F;
  ProfScope prof(kProfElementwise, s, 8.0 * double(n), 0.0);
  k_x_prep<<<grid_for(n), kT, 0, s>>>(xs, B, T_in, ld, N, F, X0, err);
  return cudaGetLastError();
}

// thread = one row r: F_out accumulators over the M blocks x NG columns (bf16 pairs), the x-part
// weight rows staged in shared memory
__global__ void k_xpart_dgrad(const __nv_bfloat16 *__restrict__ grad,
                              const __nv_bfloat16 *__restrict__ Q, int64_t mstride, int M, int NG,
                              const float *__restrict__ W, int C_in, int F_out, int64_t R,
                              float *__restrict__ out) {
  // warp = one row r: lanes stride the NG columns of each block by bf16 pairs (coalesced 128-byte
  // runs), F_out partial sums per lane, then a warp reduction
  extern __shared__ float wsm[];  // [M][F_out][NG]
  for (int i = threadIdx.x; i < M * F_out * NG; i += blockDim.x) {
    const int m = i / (F_out * NG), o = (i / NG) % F_out, j = i % NG;
    wsm[i] = W[int64_t(m * C_in + o) * NG + j];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  for (int64_t r = blockIdx.x * int64_t(wpb) + (threadIdx.x >> 5); r < R;
       r += int64_t(gridDim.x) * wpb) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int m = 0; m < M; ++m) {
      const __nv_bfloat16 *src = (m == 0 ? grad : Q + m * mstride) + r * NG;
      const float *wm = wsm + m * F_out * NG;
      for (int j = 2 * lane; j < NG; j += 64) {
        const float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(src + j));
#pragma unroll
        for (int o = 0; o < 4; ++o)
          if (o < F_out) acc[o] = fmaf(v.x, wm[o * NG + j], fmaf(v.y, wm[o * NG + j + 1], acc[o]));
      }
    }
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      float v = acc[o];
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
      if (o < F_out && lane == 0) out[r * F_out + o] += v;
    }
  }
}

cudaError_t launch_xpart_dgrad(const void *grad, const void *Q, int64_t mstride, int M, int NG,
                               const float *W, int C_in, int F_out, int64_t R, float *out,
                               cudaStream_t s) {
  if (F_out > 4 || NG % 2) return cudaErrorInvalidValue;
  ProfScope prof(kProfElementwise, s, double(R) * (2.0 * M * NG + 8.0 * F_out), 2.0 * R * M * NG * F_out);
  const int smem = M * F_out * NG * 4;
  // a plain launch: with PDL its early-resident CTAs (a full-R grid waiting on the predecessor)
  // slowed the encoder-decoder step by 9 % (11.9 K vs 10.8 K samples/s)
  const unsigned blocks = unsigned(std::min<int64_t>(ceil_div(R, kT / 32), 8 * 148));
  k_xpart_dgrad<<<blocks, kT, smem, s>>>(static_cast<const __nv_bfloat16 *>(grad),
                                             static_cast<const __nv_bfloat16 *>(Q), mstride, M,
                                             NG, W, C_in, F_out, R, out);
  return cudaGetLastError();
}

__global__ void k_bf16_to_f32(const __nv_bfloat16 *__restrict__ src, float *__restrict__ dst,
                              int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = __bfloat162float(src[i]);
}

cudaError_t launch_bf16_to_f32(const void *src, float *dst, int64_t n, cudaStream_t s) {
  k_bf16_to_f32<<<grid_for(n), kT, 0, s>>>(static_cast<const __nv_bfloat16 *>(src), dst, n);
  return cudaGetLastError();
}

cudaError_t launch_dec_input(const WindowSrc &ys, int tt, int B, int T_out, int64_t ld, int N,
                             int F, int F_out, float *out, cudaStream_t s) {
  const int64_t n = int64_t(N) * B * F_out;
  ProfScope prof(kProfElementwise, s, 8.0 * double(n), 0.0);
  k_dec_input<<<grid_for(n), kT, 0, s>>>(ys, tt, B, ld, N, F, F_out, T_out, out);
  return cudaGetLastError();
}

cudaError_t launch_loss(const float *yhat, const WindowSrc &y, int T_out, int N, int B, int F,
                        int F_out, int64_t ld, float *dyhat, double *partials, float *loss,
                        unsigned *err, cudaStream_t s) {
  ProfScope prof(kProfLoss, s, 12.0 * double(T_out) * N * B * F_out, 0.0, 2);
  cudaError_t e = pdl_launch(k_loss_partial, dim3(kLossBlocks), dim3(kT), 0, s, yhat, y, T_out,
                             N, B, F, F_out, ld, dyhat, partials);
  if (e != cudaSuccess) return e;
  return pdl_launch(k_loss_final, dim3(1), dim3(32), 0, s, static_cast<const double *>(partials),
                    kLossBlocks, int64_t(T_out) * N * B * F_out, loss, err);
}

cudaError_t launch_cand_bwd(int64_t RH, int H, const float *dHcur, const float *dHcur2,
                            const float *dy, const float *Wout, int F_out, const float *u,
                            const float *c, const float *Hprev, float *dU, float *dC,
                            float *dHprev_out, cudaStream_t s, void *dC_bf16) {
  ProfScope prof(kProfElementwise, s,
                 double(RH) * (4.0 * ((dHcur ? 1 : 0) + (dHcur2 ? 1 : 0) + 2 + (Hprev ? 1 : 0) +
                                      2 + (dHprev_out ? 1 : 0)) +
                               (dC_bf16 ? 2.0 : 0.0)), 0.0);
  k_cand_bwd<<<grid_for(RH), kT, 0, s>>>(RH, H, dHcur, dHcur2, dy, Wout, F_out, u, c, Hprev, dU,
                                         dC, dHprev_out, static_cast<__nv_bfloat16 *>(dC_bf16));
  return cudaGetLastError();
}

cudaError_t launch_cand_bwd_tc(int64_t RH, int H, const float *dHa, const float *dHb,
                               const float *dy, const float *Wout, int F_out, const float *u,
                               const void *c, const float *Hprev, float *dC, void *dCb,
                               float *dHprev, float *dG, void *dGb, cudaStream_t s) {
  if (H % 4) return cudaErrorInvalidValue;
  ProfScope prof(kProfElementwise, s,
                 double(RH) * (4.0 * ((dHa ? 1 : 0) + (dHb ? 1 : 0) + 2 + (Hprev ? 1 : 0) +
                                      (dC ? 1 : 0) + (dHprev ? 1 : 0) +
                                      (dG ? (Hprev ? 1 : 2) : 0)) +
                               2.0 * (1 + (Hprev ? 1 : 2))),
                 0.0);
  return pdl_launch(k_cand_bwd_tc, dim3(grid_for(RH / 4)), dim3(kT), 0, s, RH, H, dHa, dHb, dy,
                    Wout, F_out, u, static_cast<const __nv_bfloat16 *>(c), Hprev, dC,
                    static_cast<__nv_bfloat16 *>(dCb), dHprev, dG,
                    static_cast<__nv_bfloat16 *>(dGb));
}

cudaError_t launch_gate_bwd(int64_t RH, int H, const float *drH, const float *Hprev,
                            const float *r, const float *u, const float *dU, float *dHprev,
                            float *dG, cudaStream_t s, void *dG_bf16) {
  ProfScope prof(kProfElementwise, s,
                 double(RH) * (4.0 * (3 + (drH ? 1 : 0) + (Hprev ? 1 : 0) + (dHprev ? 2 : 0) + 2) +
                               (dG_bf16 ? 4.0 : 0.0)), 0.0);
  k_gate_bwd<<<grid_for(RH), kT, 0, s>>>(RH, H, drH, Hprev, r, u, dU, dHprev, dG,
                                         static_cast<__nv_bfloat16 *>(dG_bf16));
  return cudaGetLastError();
}

cudaError_t launch_convert_weights(const WeightJob *jobs, int njobs, cudaStream_t s) {
  if (njobs > 8) return cudaErrorInvalidValue;
  WeightParams p{};
  double n = 0;
  for (int i = 0; i < njobs; ++i) {
    p.job[i] = jobs[i];
    n += double(jobs[i].M) * jobs[i].C_in * jobs[i].Nout;
  }
  p.njobs = njobs;
  ProfScope prof(kProfElementwise, s, n * 8.0, 0.0);
  k_convert_weights<<<148 * 2, kT, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace pgti
