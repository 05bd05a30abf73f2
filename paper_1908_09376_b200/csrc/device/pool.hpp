// Process-wide pinned staging: two 64 MB pinned host buffers with one event
// each, shared by the entry sampler's chunk pipeline (sample.cu) and the
// plan's payload upload (plan.cu).  Lock `mu` for the whole use.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <mutex>

namespace midbf::dev {

struct PinnedPool {
  static constexpr size_t kBytes = size_t{64} << 20;
  std::mutex mu;
  char* h[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  void ensure();  // allocate on first use (throws CudaFailure)
};

PinnedPool& pinned_pool();

}  // namespace midbf::dev
