// K3' (fp32 SIMT) gate GEMMs of the diffusion-convolution GRU with fused epilogues (K4/K5):
//   forward  G = sum_m T_m([in, H]) W[m] + b  -> sigma / tanh / GRU update / readout
//   dgrad    dT_m = dG W[m]^T                -> split into input / hidden parts
//   wgrad    dW[m] = sum_t T_m(Z_t)^T dG_t, db = sum dG  (split-K, fixed-order reduction)
// This is the 1e-5 parity path (precision = 0).  The diffusion blocks T_m are read straight
// from the diffusion buffers (multi-source A operand), never concatenated in memory.
// Equations: Li et al. Eq. 2-3 [ext]; readings c1-c7.
#include "kernels.cuh"
#include "profile.cuh"

namespace pgti {
namespace {

constexpr int BM = 64, BK = 16, NT = 256;

__device__ __forceinline__ float sigmoidf_(float a) { return 1.0f / (1.0f + expf(-a)); }

__device__ __forceinline__ float load_a(const GconvA &a, int row, int k) {
  const int C = a.Fin + a.Hd;
  const int m = k / C;
  const int c = k - m * C;
  if (c < a.Fin) return __ldg(a.in + m * a.in_mstride + int64_t(row) * a.Fin + c);
  if (a.h) return __ldg(a.h + m * a.h_mstride + int64_t(row) * a.Hd + (c - a.Fin));
  return 0.f;
}

// ----------------------------------------------------------------------------- forward
template <int BN>
__global__ void __launch_bounds__(NT) k_gconv_fwd(const __grid_constant__ GconvFwd p) {
  constexpr int TM = 4, TN = BN / 16;
  __shared__ alignas(16) float As[BK][BM + 4];
  __shared__ alignas(16) float Bs[BK][BN];
  __shared__ float Cs[BM][BN + 1];
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  const int row0 = blockIdx.x * BM;
  const int Ktot = p.a.M * (p.a.Fin + p.a.Hd);
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < Ktot; k0 += BK) {
#pragma unroll
    for (int i = 0; i < BM * BK / NT; ++i) {
      const int e = tid + i * NT, r = e / BK, kk = e % BK;
      const int row = row0 + r, k = k0 + kk;
      As[kk][r] = (row < p.R && k < Ktot) ? load_a(p.a, row, k) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < (BK * BN + NT - 1) / NT; ++i) {
      const int e = tid + i * NT;
      if (e < BK * BN) {
        const int kk = e / BN, j = e % BN;
        Bs[kk][j] = (k0 + kk < Ktot) ? __ldg(p.W + int64_t(k0 + kk) * p.Nout + j) : 0.f;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = Bs[kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) Cs[ty * TM + i][tx * TN + j] = acc[i][j] + __ldg(p.bias + tx * TN + j);
  __syncthreads();

  if (p.mode == kEpiGate) {
    const int H = BN / 2;
    for (int e = tid; e < BM * H; e += NT) {
      const int r = e / H, j = e % H, row = row0 + r;
      if (row >= p.R) continue;
      const int64_t o = int64_t(row) * H + j;
      const float rr = sigmoidf_(Cs[r][j]), uu = sigmoidf_(Cs[r][H + j]);
      const float hp = p.Hprev ? p.Hprev[o] : 0.f;
      p.out_r[o] = rr;
      p.out_u[o] = uu;
      p.out_rH[o] = rr * hp;
    }
  } else {
    const int H = BN;
    for (int e = tid; e < BM * H; e += NT) {
      const int r = e / H, j = e % H, row = row0 + r;
      if (row >= p.R) continue;
      const int64_t o = int64_t(row) * H + j;
      const float cc = tanhf(Cs[r][j]);
      const float uu = p.u_in[o];
      const float hp = p.Hprev ? p.Hprev[o] : 0.f;
      const float hn = uu * hp + (1.0f - uu) * cc;
      p.out_c[o] = cc;
      p.out_H[o] = hn;
      Cs[r][j] = hn;
    }
    if (p.yhat) {
      __syncthreads();
      const int lane = tid & 31, w = tid >> 5;
      for (int r = w; r < BM; r += NT / 32) {
        const int row = row0 + r;
        if (row >= p.R) continue;
        for (int o = 0; o < p.F_out; ++o) {
          float s = 0.f;
          for (int j = lane; j < H; j += 32) s = fmaf(Cs[r][j], __ldg(p.Wout + j * p.F_out + o), s);
#pragma unroll
          for (int q = 16; q > 0; q >>= 1) s += __shfl_xor_sync(0xffffffffu, s, q);
          if (lane == 0) p.yhat[int64_t(row) * p.F_out + o] = s + __ldg(p.bout + o);
        }
      }
    }
  }
}

// ----------------------------------------------------------------------------- dgrad
constexpr int DBN = 64;
__global__ void __launch_bounds__(NT) k_gconv_dgrad(const __grid_constant__ GconvDgrad p) {
  constexpr int TM = 4, TN = DBN / 16;
  __shared__ alignas(16) float As[BK][BM + 4];
  __shared__ alignas(16) float Bs[BK][DBN + 4];
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  const int row0 = blockIdx.x * BM, vc0 = blockIdx.y * DBN;
  const int C = p.Fin + p.Hd, Cv = p.c_hi - p.c_lo, Vtot = p.M * Cv;
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < p.Nout; k0 += BK) {
#pragma unroll
    for (int i = 0; i < BM * BK / NT; ++i) {
      const int e = tid + i * NT, r = e / BK, kk = e % BK;
      const int row = row0 + r, k = k0 + kk;
      As[kk][r] = (row < p.R && k < p.Nout) ? __ldg(p.G + int64_t(row) * p.Nout + k) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < DBN * BK / NT; ++i) {
      const int e = tid + i * NT, v = e / BK, kk = e % BK;
      const int vc = vc0 + v, k = k0 + kk;
      float val = 0.f;
      if (vc < Vtot && k < p.Nout) {
        const int m = vc / Cv, c = p.c_lo + (vc - m * Cv);
        val = __ldg(p.W + int64_t(m * C + c) * p.Nout + k);
      }
      Bs[kk][v] = val;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = Bs[kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int row = row0 + ty * TM + i;
    if (row >= p.R) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int vc = vc0 + tx * TN + j;
      if (vc >= Vtot) continue;
      const int m = vc / Cv, c = p.c_lo + (vc - m * Cv);
      if (c < p.Fin) {
        float *d = p.Tin + m * p.tin_mstride + int64_t(row) * p.Fin + c;
        *d = p.acc_in ? *d + acc[i][j] : acc[i][j];
      } else {
        p.Th[m * p.th_mstride + int64_t(row) * p.Hd + (c - p.Fin)] = acc[i][j];
      }
    }
  }
}

// ----------------------------------------------------------------------------- wgrad
__device__ __forceinline__ float load_wa(const GconvWgrad &p, int t, int row, int vr, int C) {
  if (p.compact >= 0) {  // input rows c < compact of each block, then the bias row
    if (vr >= p.M * p.compact) return 1.0f;
    const int m = vr / p.compact, c = vr - m * p.compact;
    return __ldg(p.in + t * p.in_tstride + m * p.in_mstride + int64_t(row) * p.Fin + c);
  }
  const int m = vr / C;
  if (m >= p.M) return 1.0f;  // bias row
  const int c = vr - m * C;
  if (c < p.Fin) return __ldg(p.in + t * p.in_tstride + m * p.in_mstride + int64_t(row) * p.Fin + c);
  const int th = t + p.h_toff;
  if (!p.h || th < 0) return 0.f;
  return __ldg(p.h + th * p.h_tstride + m * p.h_mstride + int64_t(row) * p.Hd + (c - p.Fin));
}

constexpr int WKC = 2048;  // rows per split-K chunk

template <int BN>
__global__ void __launch_bounds__(NT) k_gconv_wgrad(const __grid_constant__ GconvWgrad p,
                                                    int chunks_per_t) {
  constexpr int TM = 4, TN = BN / 16;
  __shared__ alignas(16) float As[BK][BM + 4];
  __shared__ alignas(16) float Bs[BK][BN];
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  const int C = p.Fin + p.Hd, Vr = p.compact >= 0 ? p.M * p.compact + 1 : p.M * C + 1;
  const int vr0 = blockIdx.x * BM;
  const int chunk = blockIdx.y;
  const int t = chunk / chunks_per_t;
  const int rbeg = (chunk - t * chunks_per_t) * WKC;
  const int rend = min(p.R, rbeg + WKC);
  const float *G = p.G + t * p.g_tstride;
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
  for (int r0 = rbeg; r0 < rend; r0 += BK) {
#pragma unroll
    for (int i = 0; i < BM * BK / NT; ++i) {
      const int e = tid + i * NT, v = e % BM, kk = e / BM;
      const int vr = vr0 + v, row = r0 + kk;
      As[kk][v] = (vr < Vr && row < rend) ? load_wa(p, t, row, vr, C) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < (BK * BN + NT - 1) / NT; ++i) {
      const int e = tid + i * NT;
      if (e < BK * BN) {
        const int kk = e / BN, j = e % BN, row = r0 + kk;
        Bs[kk][j] = row < rend ? __ldg(G + int64_t(row) * p.Nout + j) : 0.f;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = Bs[kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  float *out = p.partial + int64_t(chunk) * Vr * p.Nout;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int vr = vr0 + ty * TM + i;
    if (vr >= Vr) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) out[int64_t(vr) * p.Nout + tx * TN + j] = acc[i][j];
  }
}

// Fixed-order sum over the split-K chunks (bitwise reproducible).
__global__ void k_reduce_chunks(const float *__restrict__ partial, int nchunks, int64_t n,
                                float *__restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < nchunks; ++c) s += partial[int64_t(c) * n + i];
    out[i] = s;
  }
}

// Same, for compact virtual rows vr -> (vr / Fs) * C_in + vr % Fs, last row -> M * C_in.
__global__ void k_reduce_compact(const float *__restrict__ partial, int nchunks, int Vr, int Nout,
                                 int Fs, int M, int C_in, float *__restrict__ out) {
  const int64_t n = int64_t(Vr) * Nout;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < nchunks; ++c) s += partial[int64_t(c) * n + i];
    const int vr = int(i / Nout), j = int(i - int64_t(vr) * Nout);
    const int row = vr >= M * Fs ? M * C_in : (vr / Fs) * C_in + vr % Fs;
    out[int64_t(row) * Nout + j] = s;
  }
}

// ----------------------------------------------------------------------------- readout wgrad
constexpr int RKC = 1024;
__global__ void __launch_bounds__(256) k_readout_wgrad(const __grid_constant__ ReadoutWgrad p,
                                                       int chunks_per_t) {
  // block: 4 row lanes x 64 column lanes; columns j in [0, H] (j == H is the bias).
  __shared__ float red[4][65 * 4];
  const int jl = threadIdx.x % 64, rl = threadIdx.x / 64;
  const int chunk = blockIdx.x, t = chunk / chunks_per_t;
  const int rbeg = (chunk - t * chunks_per_t) * RKC, rend = min(p.R, rbeg + RKC);
  const float *Hs = p.Hs + t * p.h_tstride;
  const float *dy = p.dy + int64_t(t) * p.R * p.F_out;
  const int V = p.H + 1;
  float *out = p.partial + int64_t(chunk) * V * p.F_out;
  for (int jb = 0; jb < V; jb += 64) {
    const int j = jb + jl;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    if (j < V)
      for (int row = rbeg + rl; row < rend; row += 4) {
        const float hv = j < p.H ? __ldg(Hs + int64_t(row) * p.H + j) : 1.0f;
        for (int o = 0; o < p.F_out; ++o) acc[o] = fmaf(hv, __ldg(dy + int64_t(row) * p.F_out + o), acc[o]);
      }
    for (int o = 0; o < p.F_out; ++o) red[rl][jl * 4 + o] = acc[o];
    __syncthreads();
    if (rl == 0 && j < V)
      for (int o = 0; o < p.F_out; ++o)
        out[j * p.F_out + o] = ((red[0][jl * 4 + o] + red[1][jl * 4 + o]) + red[2][jl * 4 + o]) +
                               red[3][jl * 4 + o];
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_gconv_fwd(const GconvFwd &p, cudaStream_t s) {
  const dim3 grid(unsigned(ceil_div(p.R, BM)));
  const double Kt = double(p.a.M) * (p.a.Fin + p.a.Hd), R = p.R, H = p.mode == kEpiGate ? p.Nout / 2 : p.Nout;
  // algorithmic bytes: A blocks + W + bias read once; epilogue reads Hprev (+u), writes outputs
  const double io = p.mode == kEpiGate ? (p.Hprev ? 1 : 0) + 3 : (p.Hprev ? 1 : 0) + 1 + 2;
  const double bytes = 4.0 * (R * Kt + Kt * p.Nout + p.Nout + R * H * io + (p.yhat ? R * p.F_out : 0));
  ProfScope prof(kProfGemmFwd, s, bytes, 2.0 * R * Kt * p.Nout);
  switch (p.Nout) {
    case 16: k_gconv_fwd<16><<<grid, NT, 0, s>>>(p); break;
    case 32: k_gconv_fwd<32><<<grid, NT, 0, s>>>(p); break;
    case 64: k_gconv_fwd<64><<<grid, NT, 0, s>>>(p); break;
    case 128: k_gconv_fwd<128><<<grid, NT, 0, s>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_gconv_dgrad(const GconvDgrad &p, cudaStream_t s) {
  const int Vtot = p.M * (p.c_hi - p.c_lo);
  if (Vtot <= 0) return cudaSuccess;
  const dim3 grid(unsigned(ceil_div(p.R, BM)), unsigned(ceil_div(Vtot, DBN)));
  const double R = p.R;
  const double bytes = 4.0 * (R * p.Nout + double(Vtot) * p.Nout + R * Vtot);
  ProfScope prof(kProfGemmDgrad, s, bytes, 2.0 * R * p.Nout * Vtot);
  k_gconv_dgrad<<<grid, NT, 0, s>>>(p);
  return cudaGetLastError();
}

size_t wgrad_partial_floats(int M, int C_in, int Nout, int T, int R) {
  return size_t(T) * size_t(ceil_div(R, WKC)) * size_t(M * C_in + 1) * size_t(Nout);
}

cudaError_t launch_gconv_wgrad(const GconvWgrad &p, cudaStream_t s) {
  const int C = p.Fin + p.Hd, Vr = p.compact >= 0 ? p.M * p.compact + 1 : p.M * C + 1;
  const int cpt = int(ceil_div(p.R, WKC));
  const int nchunks = p.T * cpt;
  if (int64_t(nchunks) * Vr * p.Nout > p.partial_cap) return cudaErrorInvalidValue;
  const dim3 grid(unsigned(ceil_div(Vr, BM)), unsigned(nchunks));
  const int64_t n = int64_t(Vr) * p.Nout;
  {
    const double TR = double(p.T) * p.R;
    const double bytes = 4.0 * (TR * (Vr - 1) + TR * p.Nout + double(nchunks) * n);
    ProfScope prof(kProfGemmWgrad, s, bytes, 2.0 * TR * Vr * p.Nout);
    switch (p.Nout) {
      case 16: k_gconv_wgrad<16><<<grid, NT, 0, s>>>(p, cpt); break;
      case 32: k_gconv_wgrad<32><<<grid, NT, 0, s>>>(p, cpt); break;
      case 64: k_gconv_wgrad<64><<<grid, NT, 0, s>>>(p, cpt); break;
      case 128: k_gconv_wgrad<128><<<grid, NT, 0, s>>>(p, cpt); break;
      default: return cudaErrorInvalidValue;
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ProfScope prof(kProfReduce, s, 4.0 * double(n) * (nchunks + 1), double(n) * nchunks);
  if (p.compact >= 0)
    k_reduce_compact<<<unsigned(std::min<int64_t>(ceil_div(n, 256), 1184)), 256, 0, s>>>(
        p.partial, nchunks, Vr, p.Nout, p.compact, p.M, C, p.out);
  else
    k_reduce_chunks<<<unsigned(std::min<int64_t>(ceil_div(n, 256), 1184)), 256, 0, s>>>(
        p.partial, nchunks, n, p.out);
  return cudaGetLastError();
}

size_t readout_partial_floats(int H, int F_out, int T, int R) {
  return size_t(T) * size_t(ceil_div(R, RKC)) * size_t(H + 1) * size_t(F_out);
}

cudaError_t launch_readout_wgrad(const ReadoutWgrad &p, cudaStream_t s) {
  if (p.F_out > 4) return cudaErrorInvalidValue;
  const int cpt = int(ceil_div(p.R, RKC));
  const int nchunks = p.T * cpt;
  const int64_t n = int64_t(p.H + 1) * p.F_out;
  {
    const double TR = double(p.T) * p.R;
    ProfScope prof(kProfGemmWgrad, s, 4.0 * (TR * p.H + TR * p.F_out + double(nchunks) * n),
                   2.0 * TR * n);
    k_readout_wgrad<<<unsigned(nchunks), 256, 0, s>>>(p, cpt);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ProfScope prof(kProfReduce, s, 4.0 * double(n) * (nchunks + 1), double(n) * nchunks);
  k_reduce_chunks<<<unsigned(ceil_div(n, 256)), 256, 0, s>>>(p.partial, nchunks, n, p.out);
  return cudaGetLastError();
}

}  // namespace pgti
