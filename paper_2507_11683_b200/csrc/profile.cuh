// Per-kernel-class CUDA-event timing of eager launches (bench / roofline evidence) and a
// launch counter.  Disabled by default; never records while the stream is being captured.
#pragma once

#include "common.cuh"

namespace pgti {

enum ProfClass {
  kProfGather = 0,
  kProfSpmm,
  kProfGemmFwd,
  kProfGemmDgrad,
  kProfGemmWgrad,
  kProfReduce,
  kProfElementwise,
  kProfLoss,
  kProfAdam,
  kProfIndex,
  kProfSeries,
  kProfAllreduce,
  kNumProfClasses
};

// RAII: records a start event on `s` at construction and a stop event at destruction (when
// profiling is enabled), attributing the interval and the launch's ALGORITHMIC bytes / flops
// to `cls`.  Always counts `launches` kernel launches.
class ProfScope {
 public:
  ProfScope(int cls, cudaStream_t s, double bytes, double flops, int launches = 1);
  ~ProfScope();
  ProfScope(const ProfScope &) = delete;
  ProfScope &operator=(const ProfScope &) = delete;

 private:
  int cls_;
  cudaStream_t s_;
  double bytes_, flops_;
  int slot_;
};

}  // namespace pgti
