// Thread-local error text, the sticky device error flag, pgti_check_device_error.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace {
thread_local char g_msg[1024] = "";
__device__ unsigned g_dev_err = 0;
}  // namespace

namespace pgti {

bool pdl_enabled() {
  static const bool on = [] {
    const char *v = std::getenv("PGTI_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

pgti_status fail(pgti_status st, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_msg, sizeof(g_msg), fmt, ap);
  va_end(ap);
  return st;
}

void clear_error() { g_msg[0] = 0; }

unsigned *device_error_flag() {
  static unsigned *p = nullptr;  // per process; symbol address is per device context
  void *addr = nullptr;
  if (cudaGetSymbolAddress(&addr, g_dev_err) != cudaSuccess) return nullptr;
  p = static_cast<unsigned *>(addr);
  return p;
}

}  // namespace pgti

extern "C" const char *pgti_last_error(void) { return g_msg; }

extern "C" const char *pgti_version(void) { return "libpgti 0.1 (sm_100a)"; }

extern "C" pgti_status pgti_check_device_error(void *stream) {
  cudaStream_t s = pgti::as_stream(stream);
  PGTI_CUDA_TRY(cudaStreamSynchronize(s));
  unsigned flags = 0;
  PGTI_CUDA_TRY(cudaMemcpyFromSymbol(&flags, g_dev_err, sizeof(flags)));
  unsigned zero = 0;
  PGTI_CUDA_TRY(cudaMemcpyToSymbol(g_dev_err, &zero, sizeof(zero)));
  if (flags & pgti::kDevErrRange)
    return pgti::fail(PGTI_ERR_OUT_OF_RANGE,
                      "device: a window start lay outside the series rows held by this rank");
  if (flags & pgti::kDevErrNonfinite)
    return pgti::fail(PGTI_ERR_NONFINITE, "device: non-finite loss");
  return PGTI_OK;
}
