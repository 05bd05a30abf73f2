// FP64 peaks of this B200 (MEASURED_PEAKS.json records HBM and bf16 only):
//   * DFMA throughput: every warp runs 8 independent FMA chains;
//   * DFMA latency: one dependent chain in one warp;
//   * DMMA throughput: mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64.
// Prints TFLOP/s (2 flops per FMA / per MMA multiply-add) and cycles.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) {                                                                   \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);     \
      std::exit(1);                                                                            \
    }                                                                                          \
  } while (0)

constexpr int kIters = 4096;

__global__ void dfma_tput(double* out, double a, double b) {
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

__global__ void dfma_lat(double* out, double a, double b, long long* cycles) {
  double c = threadIdx.x;
  const long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) c = fma(c, a, b);
  const long long t1 = clock64();
  if (threadIdx.x == 0) *cycles = t1 - t0;
  if (c == 1.2345) out[0] = c;
}

__global__ void dmma_tput(double* out) {
  double acc[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0;
  const double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  double* out;
  long long* cyc;
  CK(cudaMalloc(&out, 1 << 20));
  CK(cudaMalloc(&cyc, 8));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms;
  for (int warps : {4, 8, 16, 32}) {
    const int grid = sms * 2;
    dfma_tput<<<grid, warps * 32>>>(out, 0.999, 1e-3);
    CK(cudaEventRecord(e0));
    dfma_tput<<<grid, warps * 32>>>(out, 0.999, 1e-3);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double fmas = double(grid) * warps * 32 * 8 * kIters;
    std::printf("DFMA  throughput  warps/CTA=%2d grid=%d : %7.2f TFLOP/s  (%.1f FMA/cycle/SM at %d MHz)\n", warps,
                grid, 2 * fmas / (ms * 1e-3) / 1e12, fmas / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  dfma_lat<<<1, 32>>>(out, 0.999, 1e-3, cyc);
  CK(cudaDeviceSynchronize());
  long long c;
  CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
  std::printf("DFMA  latency     %.1f cycles\n", double(c) / kIters);
  for (int warps : {4, 8, 16}) {
    const int grid = sms * 2;
    dmma_tput<<<grid, warps * 32>>>(out);
    CK(cudaEventRecord(e0));
    dmma_tput<<<grid, warps * 32>>>(out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double flops = double(grid) * warps * 4 * kIters * (8.0 * 8 * 4 * 2);
    std::printf("DMMA  throughput  warps/CTA=%2d grid=%d : %7.2f TFLOP/s\n", warps, grid,
                flops / (ms * 1e-3) / 1e12);
  }
  return 0;
}
