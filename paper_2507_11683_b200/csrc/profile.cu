// Implementation of ProfScope and the pgti_profile_* / pgti_launch_count entry points.
#include <atomic>
#include <mutex>
#include <vector>

#include "profile.cuh"

namespace pgti {
namespace {

struct Rec {
  int cls;
  cudaEvent_t a, b;
  double bytes, flops;
  cudaStream_t s;
};

std::mutex g_mu;
bool g_enabled = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
std::atomic<unsigned long long> g_launches{0};

const char *kNames[kNumProfClasses] = {"gather",      "spmm",   "gemm_fwd", "gemm_dgrad",
                                       "gemm_wgrad",  "reduce", "elementwise", "loss",
                                       "adam",        "index",  "series",   "allreduce"};

cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &st) != cudaSuccess) return true;
  return st != cudaStreamCaptureStatusNone;
}

}  // namespace

ProfScope::ProfScope(int cls, cudaStream_t s, double bytes, double flops, int launches)
    : cls_(cls), s_(s), bytes_(bytes), flops_(flops), slot_(-1) {
  g_launches.fetch_add(static_cast<unsigned long long>(launches));
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_enabled || capturing(s)) return;
  Rec r{cls, get_event(), get_event(), bytes, flops, s};
  cudaEventRecord(r.a, s);
  g_recs.push_back(r);
  slot_ = int(g_recs.size()) - 1;
}

ProfScope::~ProfScope() {
  if (slot_ < 0) return;
  std::lock_guard<std::mutex> lk(g_mu);
  if (slot_ < int(g_recs.size())) cudaEventRecord(g_recs[slot_].b, s_);
}

}  // namespace pgti

using namespace pgti;

extern "C" pgti_status pgti_profile_enable(int on) {
  clear_error();
  std::lock_guard<std::mutex> lk(g_mu);
  g_enabled = on != 0;
  return PGTI_OK;
}

extern "C" int pgti_profile_num_classes(void) { return kNumProfClasses; }

extern "C" const char *pgti_profile_class_name(int c) {
  return (c >= 0 && c < kNumProfClasses) ? kNames[c] : "";
}

extern "C" pgti_status pgti_profile_read(double *ms, double *bytes, double *flops,
                                         int64_t *launches, int n) {
  clear_error();
  PGTI_REQUIRE(ms && bytes && flops && launches && n >= kNumProfClasses, PGTI_ERR_INVALID_ARG,
               "pgti_profile_read: need arrays of %d", kNumProfClasses);
  std::lock_guard<std::mutex> lk(g_mu);
  for (int i = 0; i < n; ++i) ms[i] = bytes[i] = flops[i] = 0.0, launches[i] = 0;
  pgti_status st = PGTI_OK;
  for (const Rec &r : g_recs) {
    cudaError_t e = cudaEventSynchronize(r.b);
    float t = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.a, r.b);
    if (e != cudaSuccess && st == PGTI_OK)
      st = fail(PGTI_ERR_CUDA, "pgti_profile_read: %s", cudaGetErrorString(e));
    ms[r.cls] += t;
    bytes[r.cls] += r.bytes;
    flops[r.cls] += r.flops;
    launches[r.cls] += 1;
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
  return st;
}

extern "C" pgti_status pgti_profile_timeline(int *cls, double *start_ms, double *end_ms,
                                             int64_t *stream, int cap, int *count) {
  clear_error();
  PGTI_REQUIRE(count && (cap == 0 || (cls && start_ms && end_ms && stream)), PGTI_ERR_INVALID_ARG,
               "pgti_profile_timeline: null pointer");
  std::lock_guard<std::mutex> lk(g_mu);
  *count = int(g_recs.size());
  if (g_recs.empty() || cap == 0) return PGTI_OK;
  const cudaEvent_t t0 = g_recs.front().a;
  for (int i = 0; i < int(g_recs.size()) && i < cap; ++i) {
    const Rec &r = g_recs[i];
    float a = 0.f, b = 0.f;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&a, t0, r.a);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&b, t0, r.b);
    PGTI_REQUIRE(e == cudaSuccess, PGTI_ERR_CUDA, "pgti_profile_timeline: %s",
                 cudaGetErrorString(e));
    cls[i] = r.cls, start_ms[i] = a, end_ms[i] = b;
    stream[i] = int64_t(reinterpret_cast<intptr_t>(r.s));
  }
  return PGTI_OK;
}

extern "C" uint64_t pgti_launch_count(void) { return g_launches.load(); }
