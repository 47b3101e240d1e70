// Internal launch interfaces shared by the step orchestration (dcrnn.cu) and the kernels.
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"

namespace pgti {

// ------------------------------------------------------------------ K2 CSR SpMM (diffusion)
// Y[g][n][:] = add[g][n][:] + sum_t sum_{e in row n of A_t} val_t[e] * X_t[g][col_t[e]][:]
//              (+ Y[g][n][:] if accumulate)
// Every buffer of a job is [G][N][W] with group stride gstride (floats).
struct SpmmJob {
  const int32_t *rowptr[2];
  const int32_t *col[2];
  const float *val[2];
  const float *X[2];
  int64_t nnz[2];     // entries of each term's CSR (algorithmic-byte accounting)
  int nterms;
  const float *add;   // nullable
  float *Y;
  int accumulate;
  int64_t W;
  int G;
  int64_t gstride;
  int bf16;           // X, add, Y are __nv_bfloat16 (all jobs of a launch agree)
  // Chebyshev recurrence / Clenshaw steps: Y = alpha * sum + beta * add + beta2 * add2
  // (+ Y if accumulate); the defaults (1, 1, no add2) are the plain sum, bit for bit
  float alpha = 1.f, beta = 1.f;
  const float *add2 = nullptr;
  float beta2 = 1.f;
  // shared-memory staging plan of each term's pattern (pgti_graph_windows); used when every
  // term of every job of the launch has one with the same win_rows
  const int32_t *win_ptr[2];
  const int32_t *win_nodes[2];
  const uint16_t *lcol[2];
  int win_rows, win_max;
  // filled by launch_spmm
  int64_t warp_begin, chunks;
};
constexpr int kMaxSpmmJobs = 4;
cudaError_t launch_spmm(SpmmJob *jobs, int njobs, int N, cudaStream_t s);

// ------------------------------------------------------------------ K3' fp32 SIMT GEMMs
// Virtual A operand of the diffusion convolution: row r, column k = m*C_in + c reads
//   c <  Fin : in[m*in_mstride + r*Fin + c]
//   c >= Fin : h [m*h_mstride  + r*Hd  + (c-Fin)]   (h == nullptr -> 0)
struct GconvA {
  const float *in;
  int64_t in_mstride;
  const float *h;
  int64_t h_mstride;
  int Fin, Hd, M;
};

enum EpiMode { kEpiGate = 0, kEpiCand = 1, kEpiBwd = 2 };

struct GconvFwd {
  GconvA a;
  int R;                 // rows = N*B
  const float *W;        // [M*C_in][Nout]
  const float *bias;     // [Nout]
  int Nout;              // 2H (gate) or H (cand)
  int mode;
  const float *Hprev;    // [R][H] nullable (zeros)
  // gate epilogue
  float *out_r, *out_u, *out_rH;
  // cand epilogue
  const float *u_in;
  float *out_c, *out_H;
  // optional readout yhat[R][F_out] = H' W_out + b_out
  const float *Wout, *bout;
  int F_out;
  float *yhat;
};
cudaError_t launch_gconv_fwd(const GconvFwd &p, cudaStream_t s);

// dgrad: out[r][(m,c)] = sum_j G[r][j] * W[m*C_in + c][j] for c in [c_lo, c_hi),
// written to Tin (c < Fin, layout [M][R][Fin], += if acc_in) or Th (layout [M][R][Hd]).
struct GconvDgrad {
  const float *G;   // [R][Nout]
  int R, Nout;
  const float *W;   // [M*C_in][Nout]
  int M, Fin, Hd, c_lo, c_hi;
  float *Tin;       // nullable when c_lo >= Fin
  int64_t tin_mstride;
  int acc_in;
  float *Th;
  int64_t th_mstride;
};
cudaError_t launch_gconv_dgrad(const GconvDgrad &p, cudaStream_t s);

// wgrad: dW[(m,c)][j] = sum_t sum_r A_t[r][(m,c)] * G_t[r][j]; row M*C_in = bias (A = 1).
// A_t: in part  in + t*in_tstride + m*in_mstride + r*Fin + c
//      h  part  h + (t+h_toff)*h_tstride + m*h_mstride + r*Hd + c-Fin  (t+h_toff < 0 -> 0)
struct GconvWgrad {
  const float *in;
  int64_t in_tstride, in_mstride;
  const float *h;
  int64_t h_tstride, h_mstride;
  int h_toff;
  int Fin, Hd, M;
  const float *G;        // + t*g_tstride, [R][Nout]
  int64_t g_tstride;
  int T, R, Nout;
  float *partial;        // [nchunks][M*C_in+1][Nout]
  int64_t partial_cap;   // floats available
  float *out;            // [M*C_in+1][Nout]
  // compact >= 0: compute only the input rows c < compact of every block plus the bias row
  // (virtual rows m*compact + c, then bias), written to rows m*C_in + c and M*C_in of out.
  int compact = -1;
};
cudaError_t launch_gconv_wgrad(const GconvWgrad &p, cudaStream_t s);
size_t wgrad_partial_floats(int M, int C_in, int Nout, int T, int R);

// readout wgrad: dW_out[j][o] = sum_tt sum_r Hs_tt[r][j] dy[tt][r][o], j = H -> bias
struct ReadoutWgrad {
  const float *Hs;       // + tt*h_tstride, [R][H]
  int64_t h_tstride;
  const float *dy;       // [T][R][F_out]
  int T, R, H, F_out;
  float *partial;
  float *out;            // [H+1][F_out] (W_out then b_out)
};
cudaError_t launch_readout_wgrad(const ReadoutWgrad &p, cudaStream_t s);
size_t readout_partial_floats(int H, int F_out, int T, int R);

// Skinny weight gradients: out[s][j] = sum_t sum_r S_t[r][s] * G_t[r][j] for a handful of
// "small" rows s (ns <= 12) against a wide operand G (NG <= 128 columns), split over row chunks
// with a fixed-order reduction.
//   mode kSmallBiasX : S = [x part of layer 0 (M*F values from Dx), 1]; G = dG or dCpre;
//                      row s < M*F -> out row (s/F)*C_in + s%F, s = last -> bias row M*C_in.
//   mode kSmallReadout: S = dyhat [T][R][F_out]; G = H^L_t (+ a ones column for b_out);
//                      W_out[j][o] = sum, b_out[o] = sum over the ones column.
enum SmallMode { kSmallBiasX = 0, kSmallReadout = 1 };
struct SmallWgrad {
  int mode;
  int T, R;
  const float *Dx;        // kSmallBiasX: + m*dx_mstride + t*dx_tstride + r*F + f (nullable)
  int64_t dx_mstride, dx_tstride;
  int M, F, C_in;
  const float *dy;        // kSmallReadout: [T][R][F_out]
  int F_out;
  const float *G;         // + t*g_tstride, [R][NG]
  const __nv_bfloat16 *Gb;  // same layout in bf16 (used instead of G when set)
  int64_t g_tstride;
  int NG;
  float *partial;
  int64_t partial_cap;
  float *out;             // kSmallBiasX: layer's [M*C_in+1][NG] grads block; readout: W_out
};
cudaError_t launch_small_wgrad(const SmallWgrad &p, cudaStream_t s);
size_t small_wgrad_partial_floats(int T, int R, int NG);

// ------------------------------------------------------------------ elementwise
// Where the step reads its windows: a gathered batch ([B][T][ld], idx == nullptr) or, zero-copy
// (SURVEY f2), the resident series itself by window start: sample b's row t of the slice is
// series row idx[b] - row0 + toff + t (toff = 0 for x, T_in for y).  A start whose window
// [idx[b], idx[b] + span) is not held reads zeros and raises the OUT_OF_RANGE device flag.
struct WindowSrc {
  const float *base;
  const int32_t *idx;   // nullable: gathered batch
  int64_t row0, nrows;  // series rows held (idx != nullptr)
  int toff, span;
};
cudaError_t launch_x_prep(const WindowSrc &xs, int B, int T_in, int64_t ld, int N, int F,
                          float *X0, unsigned *err, cudaStream_t s);
// encoder-decoder teacher forcing: out[n*B + b][o] = y_tt[b][n][o] for o < F_out (row tt of the
// target slice), the decoder's layer-0 input block 0
cudaError_t launch_dec_input(const WindowSrc &ys, int tt, int B, int T_out, int64_t ld, int N,
                             int F, int F_out, float *out, cudaStream_t s);
cudaError_t launch_loss(const float *yhat, const WindowSrc &ys, int T_out, int N, int B, int F,
                        int F_out, int64_t ld, float *dyhat, double *partials, float *loss,
                        unsigned *err, cudaStream_t s);
constexpr int kLossBlocks = 296;
// dH' = dHcur (+ dHcur2 if non-null) (+ dyhat W_out^T if dy non-null); dHcur nullable (= 0)
cudaError_t launch_cand_bwd(int64_t RH, int H, const float *dHcur, const float *dHcur2,
                            const float *dy,
                            const float *Wout, int F_out, const float *u, const float *c,
                            const float *Hprev, float *dU, float *dC, float *dHprev_out,
                            cudaStream_t s, void *dC_bf16 = nullptr);
// tensor-core path: candidate backward + dG_u (+ dG_r = 0 when Hprev is null), bf16 copies
// (c is bf16 on the tensor-core path)
cudaError_t launch_cand_bwd_tc(int64_t RH, int H, const float *dHa, const float *dHb,
                               const float *dy, const float *Wout, int F_out, const float *u,
                               const void *c, const float *Hprev, float *dC, void *dCb,
                               float *dHprev, float *dG, void *dGb, cudaStream_t s);
// act_dump helper: dst[i] = float(src[i]) for bf16 src
cudaError_t launch_bf16_to_f32(const void *src, float *dst, int64_t n, cudaStream_t s);
cudaError_t launch_gate_bwd(int64_t RH, int H, const float *drH, const float *Hprev,
                            const float *r, const float *u, const float *dU, float *dHprev,
                            float *dG, cudaStream_t s, void *dG_bf16 = nullptr);

// Encoder-decoder (tensor-core path): the decoder layer-0 input gradient, i.e. the F_out input
// channels of dZ = sum_m Q_m W_m^T with Q_0 = grad (bf16 [R][NG]) and Q_m = Q + m * mstride:
//   out[r][o] += sum_m sum_j Q_m[r][j] W[m*C_in + o][j]      (W fp32 [M*C_in][NG])
cudaError_t launch_xpart_dgrad(const void *grad, const void *Q, int64_t mstride, int M, int NG,
                               const float *W, int C_in, int F_out, int64_t R, float *out,
                               cudaStream_t s);

// bf16 weight tiles of the tensor-core path, rebuilt from the fp32 parameters every step:
//   fwd  (K-major B):  Wf[kb][j][c]  = W[row_kb + c][j]           c < 64, j < Nout
//   dgrad(K-major B):  Wd[v][j]      = W[(v/vseg)*C_in + coff + v%vseg][j]
struct WeightJob {
  const float *W;        // [M*C_in][Nout] fp32 (params)
  int Nout, C_in, M, Fin;
  int layer0;            // 1: blocks are the hidden part only (kb = m, rows m*C_in + Fin), then
                         //    one x k-block (kb = M): column c = m*Fin + f < M*Fin holds row
                         //    m*C_in + f (the layer-0 input channels folded into the MMA)
  void *Wf;              // bf16
  void *Wd;              // bf16
};
cudaError_t launch_convert_weights(const WeightJob *jobs, int njobs, cudaStream_t s);
// Layer-0 input channels as one 64-wide bf16 k-block per row: Xb[t][r][m*F + f] =
// bf16(Dx[m*x_mstride + t*R*F + r*F + f]) for m*F + f < M*F, zeros in the other columns.
cudaError_t launch_xpack(const float *Dx, int64_t x_mstride, int T, int64_t R, int F, int M,
                         __nv_bfloat16 *Xb, cudaStream_t s);

}  // namespace pgti
