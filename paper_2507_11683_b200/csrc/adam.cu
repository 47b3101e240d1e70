// K7: fused flat Adam (torch defaults, reading c21) with the DDP 1/R mean folded in
// (the all-reduce is a SUM, pgti_allreduce_grads).
#include <cmath>

#include "common.cuh"
#include "profile.cuh"

namespace {

__global__ void k_adam(float4 *__restrict__ p, const float4 *__restrict__ g, float4 *__restrict__ m,
                       float4 *__restrict__ v, int64_t n4, int64_t step, const int64_t *dev_step,
                       float lr, float b1, float b2, float eps, float gs) {
  pgti::griddep_launch_dependents();
  pgti::griddep_wait();
  const int64_t t = dev_step ? *dev_step + 1 : step;
  // bias corrections in double, applied once per element in fp32
  const float bc1 = float(1.0 - pow(double(b1), double(t)));
  const float rbc2 = float(1.0 / sqrt(1.0 - pow(double(b2), double(t))));
  const float step_size = lr / bc1;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4;
       i += int64_t(gridDim.x) * blockDim.x) {
    float4 pp = p[i], gg = g[i], mm = m[i], vv = v[i];
    float *pf = &pp.x, *gf = &gg.x, *mf = &mm.x, *vf = &vv.x;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float gv = gf[q] * gs;
      mf[q] = b1 * mf[q] + (1.0f - b1) * gv;
      vf[q] = b2 * vf[q] + (1.0f - b2) * gv * gv;
      pf[q] -= step_size * mf[q] / (sqrtf(vf[q]) * rbc2 + eps);
    }
    p[i] = pp, m[i] = mm, v[i] = vv;
  }
}

__global__ void k_adam_tail(float *__restrict__ p, const float *__restrict__ g,
                            float *__restrict__ m, float *__restrict__ v, int64_t lo, int64_t n,
                            int64_t step, const int64_t *dev_step, float lr, float b1, float b2,
                            float eps, float gs) {
  const int64_t t = dev_step ? *dev_step + 1 : step;
  const float bc1 = float(1.0 - pow(double(b1), double(t)));
  const float rbc2 = float(1.0 / sqrt(1.0 - pow(double(b2), double(t))));
  const int64_t i = lo + threadIdx.x;
  if (i >= n) return;
  const float gv = g[i] * gs;
  m[i] = b1 * m[i] + (1.0f - b1) * gv;
  v[i] = b2 * v[i] + (1.0f - b2) * gv * gv;
  p[i] -= (lr / bc1) * m[i] / (sqrtf(v[i]) * rbc2 + eps);
}

__global__ void k_incr(int64_t *c) { *c += 1; }

}  // namespace

extern "C" pgti_status pgti_adam_step(float *params, const float *grads, float *m, float *v,
                                      size_t n, int64_t step, int64_t *dev_step, float lr,
                                      float beta1, float beta2, float eps, float grad_scale,
                                      void *stream) {
  pgti::clear_error();
  PGTI_REQUIRE(params && grads && m && v, PGTI_ERR_INVALID_ARG, "pgti_adam_step: null pointer");
  PGTI_REQUIRE(step > 0 || dev_step, PGTI_ERR_INVALID_ARG,
               "pgti_adam_step: step <= 0 needs dev_step");
  PGTI_REQUIRE(pgti::aligned16(params) && pgti::aligned16(grads) && pgti::aligned16(m) &&
                   pgti::aligned16(v),
               PGTI_ERR_ALIGNMENT, "pgti_adam_step: buffers must be 16-byte aligned");
  PGTI_REQUIRE(std::isfinite(lr) && beta1 >= 0 && beta1 < 1 && beta2 >= 0 && beta2 < 1 && eps > 0,
               PGTI_ERR_INVALID_ARG, "pgti_adam_step: lr=%g beta1=%g beta2=%g eps=%g", lr, beta1,
               beta2, eps);
  cudaStream_t s = pgti::as_stream(stream);
  const int64_t *ds = step > 0 ? nullptr : dev_step;
  const int64_t n4 = int64_t(n) / 4;
  // algorithmic bytes: read params, grads, m, v; write params, m, v
  pgti::ProfScope prof(pgti::kProfAdam, s, 28.0 * double(n), 10.0 * double(n),
                       (n4 > 0) + (int64_t(n) > n4 * 4) + (ds != nullptr));
  if (n4 > 0) {
    const int grid = int(std::min<int64_t>(pgti::ceil_div(n4, 256), 148 * 8));
    PGTI_CUDA_TRY(pgti::pdl_launch(k_adam, dim3(grid), dim3(256), 0, s,
                                   reinterpret_cast<float4 *>(params),
                                   reinterpret_cast<const float4 *>(grads),
                                   reinterpret_cast<float4 *>(m), reinterpret_cast<float4 *>(v), n4,
                                   step, ds, lr, beta1, beta2, eps, grad_scale));
  }
  if (int64_t(n) > n4 * 4) {
    k_adam_tail<<<1, 32, 0, s>>>(params, grads, m, v, n4 * 4, int64_t(n), step, ds, lr, beta1,
                                 beta2, eps, grad_scale);
    PGTI_LAUNCH_TRY();
  }
  if (ds) {
    k_incr<<<1, 1, 0, s>>>(dev_step);
    PGTI_LAUNCH_TRY();
  }
  return PGTI_OK;
}
