// Fixed cost of launching a k1_flow-shaped kernel: back-to-back launches of an
// (almost) empty kernel with the same grid / block / dynamic shared memory /
// parameter size, cooperative or not, plain or captured in a graph.
#include <cuda_runtime.h>

#include <cstdio>

struct Params {
  char pad[2800];
};

__global__ void __launch_bounds__(384, 1) empty_kernel(const __grid_constant__ Params p, int* out) {
  extern __shared__ unsigned char sm[];
  if (threadIdx.x == 0 && p.pad[0] == 7) out[blockIdx.x] = sm[0];
}

#define CK(x)                                                            \
  do {                                                                   \
    cudaError_t e_ = (x);                                                \
    if (e_ != cudaSuccess) {                                             \
      std::printf("%s: %s\n", #x, cudaGetErrorString(e_));              \
      return 1;                                                          \
    }                                                                    \
  } while (0)

int main() {
  int* out;
  CK(cudaMalloc(&out, 4096));
  const size_t smems[3] = {0, 100 << 10, 213 << 10};
  for (size_t smem : smems) {
    CK(cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    for (int coop = 0; coop < 2; ++coop) {
      Params p{};
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(384);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = coop;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaStream_t s;
      CK(cudaStreamCreate(&s));
      cfg.stream = s;
      for (int i = 0; i < 10; ++i) CK(cudaLaunchKernelEx(&cfg, empty_kernel, p, out));
      cudaEvent_t a, b;
      CK(cudaEventCreate(&a));
      CK(cudaEventCreate(&b));
      const int n = 200;
      CK(cudaEventRecord(a, s));
      for (int i = 0; i < n; ++i) CK(cudaLaunchKernelEx(&cfg, empty_kernel, p, out));
      CK(cudaEventRecord(b, s));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      // graph of one launch, replayed
      cudaGraph_t g;
      cudaGraphExec_t ge;
      CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      CK(cudaLaunchKernelEx(&cfg, empty_kernel, p, out));
      CK(cudaStreamEndCapture(s, &g));
      CK(cudaGraphInstantiate(&ge, g, 0));
      for (int i = 0; i < 10; ++i) CK(cudaGraphLaunch(ge, s));
      CK(cudaEventRecord(a, s));
      for (int i = 0; i < n; ++i) CK(cudaGraphLaunch(ge, s));
      CK(cudaEventRecord(b, s));
      CK(cudaEventSynchronize(b));
      float msg;
      CK(cudaEventElapsedTime(&msg, a, b));
      std::printf("smem %3zu KB cooperative %d: %.2f us per launch, %.2f us per graph replay\n", smem >> 10, coop,
                  ms * 1e3 / n, msg * 1e3 / n);
    }
  }
  return 0;
}
