// Microbenchmark (dev tool, not a test): per-kernel cost of a dependent chain of small kernels
// captured in a CUDA graph, plain stream order vs programmatic dependent launch (PDL:
// griddepcontrol.launch_dependents at kernel start + griddepcontrol.wait before touching data).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tests/cuda/pdl_mb.cu -o /tmp/pdl
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("%s failed: %s\n", #x, cudaGetErrorString(e));                      \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

template <bool PDL>
__global__ void k_step(float *buf, int n, int iters) {
  if (PDL) asm volatile("griddepcontrol.launch_dependents;");
  __shared__ float s[1024];
  s[threadIdx.x] = 0.f;  // prologue work that does not touch dependent data
  if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    float v = buf[i];
    for (int k = 0; k < iters; ++k) v = v * 0.999f + 0.001f;
    buf[i] = v + s[threadIdx.x];
  }
}

int main() {
  float *buf;
  const int n_max = 148 * 8 * 256;
  CK(cudaMalloc(&buf, n_max * 4));
  CK(cudaMemset(buf, 0, n_max * 4));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  cudaEventCreate(&a), cudaEventCreate(&b);
  const int chain = 200;
  for (int blocks : {104, 296, 1184}) {
    for (int iters : {0, 200}) {
      for (int pdl = 0; pdl < 2; ++pdl) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
        for (int k = 0; k < chain; ++k) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(blocks), cfg.blockDim = dim3(256), cfg.stream = s;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at, cfg.numAttrs = pdl ? 1 : 0;
          if (pdl)
            CK(cudaLaunchKernelEx(&cfg, k_step<true>, buf, blocks * 256, iters));
          else
            CK(cudaLaunchKernelEx(&cfg, k_step<false>, buf, blocks * 256, iters));
        }
        CK(cudaStreamEndCapture(s, &g));
        CK(cudaGraphInstantiate(&ge, g, 0));
        for (int w = 0; w < 3; ++w) CK(cudaGraphLaunch(ge, s));
        CK(cudaStreamSynchronize(s));
        cudaEventRecord(a, s);
        for (int w = 0; w < 10; ++w) CK(cudaGraphLaunch(ge, s));
        cudaEventRecord(b, s);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("blocks=%5d iters=%4d %-6s %7.2f us/kernel\n", blocks, iters, pdl ? "PDL" : "plain",
               ms * 1000 / (10 * chain));
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
      }
    }
  }
  return 0;
}
