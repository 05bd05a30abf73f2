// Read-bandwidth probe for the K1 design space on B200 (sm_100a): how fast
// can one SM-resident kernel stream a large read-only buffer with
//   (a) per-warp rings of cp.async.bulk (TMA bulk) copies into shared memory,
//       varying chunk size / ring depth / warps per CTA, and
//   (b) plain coalesced 128-bit / 256-bit global loads with unrolling?
// Usage: bw_probe [MB]   (prints one line per configuration, GB/s).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <algorithm>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                              \
    }                                                                            \
  } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// Each warp streams its own contiguous share of the buffer in `chunk`-byte
// bulk copies through a `depth`-slot ring; lane 0 issues, the warp waits on
// the slot barrier and touches one word so the data is consumed.
// mode 0: warp streams one contiguous share; mode > 0: strips of `mode`
// consecutive chunks dealt round-robin over the warps (K1's strip deal).
__global__ void tma_stream(const char* __restrict__ buf, size_t bytes, int chunk, int depth, double* sink, int misalign,
                           int mode) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned char* ring = smem + size_t(w) * depth * chunk;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(nw) * depth * chunk) + w * depth;
  if (lane == 0)
    for (int s = 0; s < depth; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const size_t gw = size_t(blockIdx.x) * nw + w, NW = size_t(gridDim.x) * nw;
  const size_t nchunks = bytes / chunk;
  size_t per = (nchunks + NW - 1) / NW;
  size_t c0 = gw * per, c1 = c0 + per < nchunks ? c0 + per : nchunks;
  if (mode > 0) {  // my k-th chunk -> global chunk of strip (gw + (k/mode)*NW), offset k%mode
    const size_t nstrip = nchunks / mode;
    const size_t mine = gw < nstrip ? (nstrip - 1 - gw) / NW + 1 : 0;
    c0 = 0;
    c1 = mine * mode;
  }
  auto gchunk = [&](size_t k) -> size_t {
    return mode > 0 ? (gw + (k / mode) * NW) * mode + (k % mode) : k;
  };
  double acc = 0;
  size_t issued = c0;
  auto issue = [&](size_t c) {
    const unsigned slot = (c - c0) % depth;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[slot])), "r"(chunk)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            sa(ring + size_t(slot) * chunk)),
        "l"(buf + gchunk(c) * chunk + misalign), "r"(chunk), "r"(sa(&bars[slot]))
        : "memory");
  };
  if (lane == 0)
    for (; issued < c1 && issued < c0 + depth; ++issued) issue(issued);
  for (size_t c = c0; c < c1; ++c) {
    const unsigned slot = (c - c0) % depth, par = ((c - c0) / depth) & 1;
    asm volatile(
        "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
            sa(&bars[slot])),
        "r"(par)
        : "memory");
    acc += reinterpret_cast<const double*>(ring + size_t(slot) * chunk)[lane];
    __syncwarp();
    if (lane == 0 && issued < c1) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(issued++);
    }
  }
  if (acc == 12345.678) *sink = acc;
}

template <int U>
__global__ void ldg_stream(const double2* __restrict__ buf, size_t n, double* sink) {
  const size_t tid = size_t(blockIdx.x) * blockDim.x + threadIdx.x, T = size_t(gridDim.x) * blockDim.x;
  double acc = 0;
  size_t i = tid;
  for (; i + (U - 1) * T < n; i += U * T) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(buf + i + u * T);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
  }
  for (; i < n; i += T) acc += __ldcs(buf + i).x;
  if (acc == 12345.678) *sink = acc;
}

int main(int argc, char** argv) {
  const size_t mb = argc > 1 ? std::atoll(argv[1]) : 1024;
  const size_t bytes = mb << 20;
  char* buf;
  double* sink;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(buf, 1, bytes));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  struct Cfg {
    int warps, chunk, depth, ctas_per_sm;
  } cfgs[] = {{4, 16384, 3, 1}, {8, 8192, 3, 1}};
  for (size_t sz : {std::min(size_t(358) << 20, bytes), bytes}) {
    for (int mode : {0, 3, 4}) {
      for (int coop : {0, 1}) {
        for (const Cfg& c : cfgs) {
          const size_t smem = size_t(c.warps) * c.depth * c.chunk + size_t(c.warps) * c.depth * 8;
          const int grid = sms * c.ctas_per_sm;
          cudaLaunchConfig_t lc = {};
          lc.gridDim = dim3(grid);
          lc.blockDim = dim3(c.warps * 32);
          lc.dynamicSmemBytes = smem;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeCooperative;
          at[0].val.cooperative = coop;
          lc.attrs = at;
          lc.numAttrs = 1;
          for (int it = 0; it < 2; ++it) CK(cudaLaunchKernelEx(&lc, tma_stream, (const char*)buf, sz, c.chunk, c.depth, sink, 0, mode));
          CK(cudaEventRecord(a));
          const int reps = 20;
          for (int it = 0; it < reps; ++it) CK(cudaLaunchKernelEx(&lc, tma_stream, (const char*)buf, sz, c.chunk, c.depth, sink, 0, mode));
          CK(cudaEventRecord(b));
          CK(cudaEventSynchronize(b));
          float ms;
          CK(cudaEventElapsedTime(&ms, a, b));
          std::printf("tma size=%5zu MB mode=%d coop=%d warps=%2d chunk=%6d depth=%d : %7.1f GB/s  %7.1f us/launch\n",
                      sz >> 20, mode, coop, c.warps, c.chunk, c.depth, double(sz) * reps / (ms * 1e-3) / 1e9,
                      ms * 1e3 / reps);
        }
      }
    }
  }
  const size_t n = bytes / 16;
  for (int tpb : {512}) {
    for (int mult : {2}) {
      const int grid = sms * mult;
      auto run = [&](auto kern, const char* name) {
        for (int it = 0; it < 2; ++it) kern<<<grid, tpb>>>(reinterpret_cast<double2*>(buf), n, sink);
        CK(cudaEventRecord(a));
        for (int it = 0; it < 10; ++it) kern<<<grid, tpb>>>(reinterpret_cast<double2*>(buf), n, sink);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        std::printf("ldg  %s tpb=%4d grid=%4d : %7.1f GB/s\n", name, tpb, grid, double(bytes) * 10 / (ms * 1e-3) / 1e9);
      };
      run(ldg_stream<4>, "U4");
      run(ldg_stream<8>, "U8");
    }
  }
  return 0;
}
