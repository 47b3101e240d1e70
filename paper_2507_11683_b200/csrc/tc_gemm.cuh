// Host interfaces of the tcgen05 (bf16 -> fp32 TMEM) gate GEMMs of the precision = 1 path.
// All diffusion blocks handled here are 64 channels wide (hidden state H = 64, or the 64-wide
// input of layer > 0): one 128-byte SWIZZLE_128B row per row of A, so one k-block = one block.
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"

namespace pgti {

constexpr int kTcC = 64;  // channels per k-block

// Forward gate / candidate GEMM with fused GRU epilogue (K3 + K4 + K5).
//   G[r][j] = sum_kb A_kb[r][0:64] . Wf[kb][j][0:64] + bias[j] (+ layer-0 x part by FFMA)
struct TcFwd {
  int R, H, Nout, mode;             // mode: kEpiGate / kEpiCand (kernels.cuh)
  const __nv_bfloat16 *A_in;        // [M][R][64] (layer > 0 input blocks) or null
  const __nv_bfloat16 *A_h;         // [M][R][64] hidden blocks (H_{t-1} or r*H) or null (= 0)
  int M;
  const __nv_bfloat16 *Wf;          // [nkb_total][Nout][64]: K-major B tiles
  int nkb_total;
  int nkb;                          // active k-blocks
  signed char kb_src[16], kb_m[16], kb_w[16];
  const float *bias;
  // layer-0 x part (fp32, FFMA): Dx[m*dx_mstride + r*F + f] * Wx[(m*C_in + f)*Nout + j]
  const float *Dx;
  int64_t dx_mstride;
  int F, C_in;
  const float *Wx;
  const float *Hprev;               // fp32 [R][H] or null
  float *out_r, *out_u;             // gate
  __nv_bfloat16 *out_rH;            // gate: r*Hprev in bf16 (block 0 of the r*H diffusion)
  const float *u_in;                // cand
  float *out_c, *out_H;
  __nv_bfloat16 *out_Hb;
  const float *Wout, *bout;
  int F_out;
  float *yhat;
};
cudaError_t launch_tc_fwd(const TcFwd &p, cudaStream_t s);

// dgrad: dT[r][v] = sum_j G[r][j] Wd[v][j]; v -> (m, c) = (v / vseg, coff + v % vseg);
// c < Fin -> Tin[m][r][c] (+= if acc_in), else Th[m][r][c - Fin]   (fp32 outputs)
struct TcDgrad {
  const __nv_bfloat16 *G;           // [R][Nout]
  int R, Nout;
  const __nv_bfloat16 *Wd;          // [V][Nout]
  int V, vseg, coff, Fin, Hd;
  float *Tin;
  int64_t tin_mstride;
  int acc_in;
  float *Th;
  int64_t th_mstride;
};
cudaError_t launch_tc_dgrad(const TcDgrad &p, cudaStream_t s);

// wgrad: partial[chunk][v][j] = sum_{rows of chunk} A[v][row] G_t[row][j], then a fixed-order
// reduction over chunks into out rows (v / vseg) * C_in + coff + v % vseg.
//   v in tile of 128 = two 64-channel chunks; layout "pairs" (vseg = 128): chunk q of tile i is
//   source q (0 = in, 1 = h) of block m = i; layout "h only" (vseg = 64): chunk q is block
//   2 i + q of the h source.
struct TcWgrad {
  const __nv_bfloat16 *A_in;        // [T][M][R][64] or null
  const __nv_bfloat16 *A_h;         // [T][M][R][64]
  int h_toff;                       // h source at t + h_toff (< 0 -> zeros)
  int T, M, R;
  const __nv_bfloat16 *G;           // [T][R][Nout]
  int Nout;
  int V, vseg, coff, C_in;
  float *partial;
  int64_t partial_cap;
  float *out;                       // layer's [M*C_in + 1][Nout] block of grads
};
cudaError_t launch_tc_wgrad(const TcWgrad &p, cudaStream_t s);
size_t tc_wgrad_partial_floats(int V, int Nout, int T, int R);

}  // namespace pgti
