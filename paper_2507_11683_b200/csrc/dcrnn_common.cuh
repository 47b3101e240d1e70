// Shared pieces of the step orchestration (dcrnn.cu: fp32 path + C ABI; dcrnn_tc.cu: bf16
// tcgen05 path): dimensions, parameter offsets, descriptor checks, diffusion launch helpers.
#pragma once

#include <vector>

#include "kernels.cuh"

namespace pgti {
namespace detail {

struct Dims {
  int N, F, F_out, L, H, K, T_in, T_out, B, M;
  int64_t R, ld;
  int precision;
  int model;    // 0 stepwise stack, 1 encoder-decoder (pgti.h)
  int teacher;  // encoder-decoder: bit s-1 set = decoder step s is fed the previous target
  // decoder step s >= 1 fed the target y_{s-1} (else its own prediction yhat_{s-1})
  bool fed_truth(int s) const { return s >= 1 && ((teacher >> (s - 1)) & 1); }
  int cheb;     // diffusion blocks by the Chebyshev recurrence (reading c25)
  // hidden-state steps: T_in (stepwise) or T_in + T_out (encoder then decoder)
  int steps() const { return T_in + (model ? T_out : 0); }
};

// parameter offsets (floats) in the flat layout of pgti.h; layer sets: [0, L) the (encoder)
// stack, [L, 2L) the decoder of model 1
struct ParamOffsets {
  std::vector<size_t> Wru, bru, Wc, bc;
  size_t Wout, bout, total;
};

ParamOffsets param_offsets(const Dims &d);
pgti_status check_desc(const pgti_dcrnn_desc *desc, Dims *out);

// Forward diffusion: blocks base + m*mstride (block 0 given, or src0 when non-null), G groups of
// stride gstride, width W.  transposed = 1 uses P_f^T / P_b^T; bf16 = 1: blocks are bf16.
cudaError_t diffuse_fwd(const pgti_dcrnn_desc &g, const Dims &d, float *base, int64_t mstride,
                        int G, int64_t gstride, int64_t W, cudaStream_t s, int bf16 = 0,
                        int transposed = 0, const void *src0 = nullptr);

// Adjoint of the diffusion features (Horner form):
//   out (+)= dT_0 + P_f^T (dT_1 + P_f^T (... + P_f^T dT_K)) + P_b^T (dT_{K+1} + ... P_b^T dT_2K)
struct AdjChain {
  const float *dT;
  int64_t mstride, W;
  float *out;
  int accumulate;
  float *tf[2], *tb[2];
};
cudaError_t diffuse_adj(const pgti_dcrnn_desc &g, const Dims &d, AdjChain *ch, int nch,
                        cudaStream_t s);

// precision = 1 (dcrnn_tc.cu)
size_t workspace_tc(const Dims &d);
pgti_status run_step_tc(const pgti_dcrnn_desc &g, const Dims &d, const float *params,
                        float *grads, const WindowSrc &x, const WindowSrc &y, float *loss_dev,
                        char *ws, float *act_dump, cudaStream_t s);

}  // namespace detail
}  // namespace pgti

#define CU(expr)                                                                                \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      return ::pgti::fail(PGTI_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_),     \
                          __FILE__, __LINE__);                                                  \
  } while (0)
