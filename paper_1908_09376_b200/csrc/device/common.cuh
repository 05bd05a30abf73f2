// Device-side helpers shared by the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../status.hpp"

// Checked builds (make checked -> libmidbf_b200_checked.so, -DMIDBF_CHECKED):
// device-side bounds assertions on every table-driven access of the apply
// kernels (arena ranges of the panel copies, stage-buffer / output indices,
// shared-memory slot sizes).  A violation prints its site and traps, which
// fails the launch with an error instead of reading or writing out of
// bounds.  This pool closes compute-sanitizer, so the checked build run over
// the small parity cases (tests/test_gpu_checked.py) stands in for memcheck.
#ifdef MIDBF_CHECKED
#include <cstdio>
#define MIDBF_DCHECK(cond, what)                                                                       \
  do {                                                                                                 \
    if (!(cond)) {                                                                                     \
      printf("MIDBF_CHECKED violation: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,     \
             static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                              \
      __trap();                                                                                        \
    }                                                                                                  \
  } while (0)
#else
#define MIDBF_DCHECK(cond, what) \
  do {                           \
  } while (0)
#endif

namespace midbf::dev {

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw detail::CudaFailure(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// Fails loudly when no sm_100 device is present: there is no CPU fallback.
int require_device();

// Programmatic dependent launch (PTX griddepcontrol, sm_90+): a stage may
// start its factor-data prefetch while the previous stage drains, and waits
// here before touching the previous stage's output vector.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// One bulk L2 prefetch of a contiguous global range (TMA unit, no SM
// registers or shared memory involved).  `bytes` must be a multiple of 16.
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

}  // namespace midbf::dev
