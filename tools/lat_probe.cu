// DFMA dependent-chain latency and LDS.128 latency on the device (one warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b) {
  __shared__ double2 sm[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = make_double2(i, 0);
  __syncwarp();
  double x = a;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a); x = fma(x, b, a);
  }
  long long t1 = clock64();
  int idx = threadIdx.x;
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    double2 v = sm[idx];
    idx = (static_cast<int>(v.x) + 1) & 1023;
  }
  long long t3 = clock64();
  // independent DFMA throughput, one warp: 8 chains
  double y[8];
  for (int j = 0; j < 8; ++j) y[j] = a + j;
  long long t4 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) y[j] = fma(y[j], b, a);
  }
  long long t5 = clock64();
  double s = x + idx;
  for (int j = 0; j < 8; ++j) s += y[j];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / 4096;
    cyc[1] = (t3 - t2) / 1024;
    cyc[2] = (t5 - t4) * 100 / 8192;
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMallocManaged(&c, 64);
  k<<<1, 32>>>(o, c, 1e-3, 0.999); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1e-3, 0.999); cudaDeviceSynchronize();
  printf("DFMA dependent latency %lld cycles; LDS.128 dependent latency %lld cycles; independent DFMA issue %.2f cycles/warp-instr\n", c[0], c[1], c[2] / 100.0);
}
