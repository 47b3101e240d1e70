// Host interfaces of the tcgen05 (bf16 -> fp32 TMEM) gate GEMMs of the precision = 1 path.
// All diffusion blocks handled here are 64-channel slices (hidden state H = 64, the 64-wide
// input of layer > 0, or 64-column slices of the diffused gradients): one 128-byte
// SWIZZLE_128B row per row of A, so one k-block = one 64-channel slice of one block.
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"

namespace pgti {

constexpr int kTcC = 64;   // channels per k-block
constexpr int kTcMaxKb = 16;

// Multi-block GEMM with a fused epilogue, one CTA per (128 rows, 64-column tile):
//   acc[r][n] = sum_kb A_kb[r][0:64] . B_kb[n][0:64]
// A_kb = slice kb_ac of block kb_am of operand map kb_as (0: A0, 1: A1), each [blocks][R][CA].
// B_kb = rows (kb_by + 64*tile) and columns kb_bx of the 3-D bf16 map Bw ([Z][Y][X]) at z=kb_bz.
// Epilogues (mode):
//   kEpiGate: gate = acc + bias (+ layer-0 x part by FFMA); tile 0 -> r = sigma(.), writes r
//             and r*H_{t-1} (bf16); tile 1 -> u = sigma(.).
//   kEpiCand: c = tanh(acc + bias + x part); H_t = u H_{t-1} + (1-u) c (fp32 and bf16);
//             optional readout yhat = H_t W_out + b_out.
//   kEpiBwd : dst[tile][r][0:64] (+)= acc  (the adjoint-diffused gradient, fp32).
struct TcFwd {
  int R, H, Nout, mode, ntiles;
  const __nv_bfloat16 *A0, *A1;     // [blocks][R][CA] (null -> unused)
  int CA, M0, M1;                   // channels per row of A0/A1; block counts
  const __nv_bfloat16 *Bw;          // bf16 weights viewed as [Z][Y][X] (X contiguous)
  int bX, bY, bZ;
  int nkb;
  signed char kb_as[kTcMaxKb], kb_am[kTcMaxKb], kb_ac[kTcMaxKb];
  short kb_bx[kTcMaxKb], kb_by[kTcMaxKb], kb_bz[kTcMaxKb];
  const float *bias;
  // layer-0 x part (fp32, FFMA): Dx[m*dx_mstride + r*F + f] * Wx[(m*C_in + f)*Nout + j]
  const float *Dx;
  int64_t dx_mstride;
  int F, C_in, M;
  const float *Wx;
  const float *Hprev;               // fp32 [R][H] or null
  __nv_bfloat16 *out_r;             // gate: r (bf16: read only by the backward)
  float *out_u;                     // gate: u (fp32: the forward recurrence reads it)
  __nv_bfloat16 *out_rH;            // gate: r*Hprev in bf16 (block 0 of the r*H diffusion)
  const float *u_in;                // cand
  __nv_bfloat16 *out_c;             // cand: c (bf16: read only by the backward)
  float *out_H;
  __nv_bfloat16 *out_Hb;
  const float *Wout, *bout;
  int F_out;
  float *yhat;
  float *dst[2];                    // bwd
  int dst_acc[2];
  // bwd, candidate GEMM: column tile `fuse_tile` is d(r*H_{t-1}); instead of storing it, run the
  // gate backward there: dG_r = acc H_{t-1} r (1-r) (fp32 g_dG + bf16 g_dGb, [R][2H], columns
  // [0,H)), g_dHprev += acc r.  Uses Hprev.  -1 = off.  g_dG may be null (bf16 copy only).
  int fuse_tile = -1;
  // set by launch_tc_fwd: 1 = libm tanhf / expf activations, 0 = MUFU tanh (default)
  int exact = 0;
  const __nv_bfloat16 *g_r;
  float *g_dG;
  __nv_bfloat16 *g_dGb;
  float *g_dHprev;
};
cudaError_t launch_tc_fwd(const TcFwd &p, cudaStream_t s);

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
  // layer 0 ("h only", vseg = 64) with x_F > 0: the packed input rows Xb [T][R][64] (A_in,
  // one block) are chunk M of the v range, i.e. V = (M + 1) 64, and their reduced rows
  // v = M*64 + m*x_F + f (< M*x_F) go to grads rows m*C_in + f (the layer-0 input part)
  int x_F = 0;
  // with x_F: packed channel M*x_F is the constant 1 (k_xpack), its reduced row is the layer's
  // bias gradient (grads row M*C_in)
  int x_bias = 0;
};
cudaError_t launch_tc_wgrad(const TcWgrad &p, cudaStream_t s);
size_t tc_wgrad_partial_floats(int V, int Nout, int T, int R);

}  // namespace pgti
