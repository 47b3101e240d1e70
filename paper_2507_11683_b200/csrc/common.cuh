// Shared host/device helpers of libpgti (error plumbing, launch helpers, small math).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstddef>

#include "pgti.h"

namespace pgti {

// Records `st` with a printf-style message in the thread-local error buffer and returns it.
pgti_status fail(pgti_status st, const char *fmt, ...);
void clear_error();
// Device address of the sticky error-flag word (bit 1: out of range, bit 2: non-finite).
unsigned *device_error_flag();
// internal view of a series handle (series.cu)
void series_view(const pgti_series *sr, const float **buf, int64_t *row0, int64_t *nrows,
                 int64_t *N, int64_t *F, int64_t *ld);

enum : unsigned { kDevErrRange = 1u, kDevErrNonfinite = 2u };

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }
inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

constexpr int kNumSMs = 148;  // B200

// Programmatic dependent launch (PDL).  Kernels launched with pdl_launch may start while their
// stream predecessor is still finishing: they run their data-independent prologue, then
// griddep_wait() (griddepcontrol.wait: every prerequisite grid has completed and its writes are
// visible) before touching any input; griddep_launch_dependents() lets the successor's CTAs be
// scheduled once every CTA of this grid has started.  Both are no-ops for normal launches.
// PGTI_PDL=0 turns PDL off (A/B measurements).
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();
template <typename K, typename... Args>
cudaError_t pdl_launch(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid, cfg.blockDim = block, cfg.dynamicSmemBytes = smem, cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at, cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args...);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace pgti

#define PGTI_REQUIRE(cond, status, ...)                     \
  do {                                                      \
    if (!(cond)) return ::pgti::fail((status), __VA_ARGS__); \
  } while (0)

#define PGTI_CUDA_TRY(call)                                                                 \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return ::pgti::fail(PGTI_ERR_CUDA, "%s failed: %s (%s:%d)", #call,                   \
                          cudaGetErrorString(e_), __FILE__, __LINE__);                      \
  } while (0)

#define PGTI_LAUNCH_TRY() PGTI_CUDA_TRY(cudaGetLastError())

#define PGTI_STATUS_TRY(expr)              \
  do {                                     \
    pgti_status s_ = (expr);               \
    if (s_ != PGTI_OK) return s_;          \
  } while (0)
