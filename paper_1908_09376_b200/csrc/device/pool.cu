#include "pool.hpp"

#include "common.cuh"

namespace midbf::dev {

void PinnedPool::ensure() {
  if (h[0]) return;
  for (int b = 0; b < 2; ++b) {
    cuda_check(cudaMallocHost(&h[b], kBytes), "cudaMallocHost staging buffer");
    cuda_check(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming), "event");
  }
}

PinnedPool& pinned_pool() {
  static PinnedPool* p = new PinnedPool;  // never destroyed (CUDA teardown order)
  return *p;
}

}  // namespace midbf::dev
