// Kernel descriptions for K(x, xi) = exp(2*pi*i*Phi(x, xi)).
//
// The reference passes a per-entry std::function (include/midbf/butterfly.hpp:24)
// built from the phase functions of src/kernels.cpp:18-35 and the low-rank
// phase of src/metrics.cpp:18-24.  A device sampler cannot call a host
// std::function, so the B200 build names the phase in a plain struct that the
// GPU evaluates directly (the C layout is `midbf_kernel_desc` in
// include/midbf_b200.h).
#pragma once

#include "midbf/types.hpp"

extern "C" {
#include "midbf_b200.h"
}

namespace midbf::ker {

enum class Kind : int {
  Fio2D = MIDBF_KERNEL_FIO2D,      // x.xi + sqrt(c1(x)^2 xi1^2 + c2(x)^2 xi2^2)  (src/kernels.cpp:18-24)
  Fio3D = MIDBF_KERNEL_FIO3D,      // 3D extension of the above (BASELINE.json configs[3])
  LowRank = MIDBF_KERNEL_LOWRANK,  // Phi = A(i,:) . B(j,:), A,B real N x r  (src/metrics.cpp:18-24)
  Nufft = MIDBF_KERNEL_NUFFT,      // Phi = x . xi  (src/kernels.cpp:26-29)
  Const = MIDBF_KERNEL_CONST,      // test kernel: K = c
  Rank1 = MIDBF_KERNEL_RANK1,      // test kernel: K = u(i) v(j)
};

using KernelDesc = midbf_kernel_desc;

// x.xi + sqrt(c1^2 xi1^2 + c2^2 xi2^2), c1 = (2 + sin(2 pi x1) sin(2 pi x2))/16,
// c2 = (2 + cos(2 pi x1) cos(2 pi x2))/16  (src/kernels.cpp:18-24).
double fio2d_phase(const double* x, const double* xi);
// The 3D phase of BASELINE.json configs[3]; not present in the reference.
double fio3d_phase(const double* x, const double* xi);

// Row-major n x n grid, point i*n+j at (i/n, j/n) (src/kernels.cpp:37-45).
MatXd grid2d(Index n);

// Host entry evaluator equivalent to the descriptor (used by the EntryFn
// path and by metrics on the host).
Cplx entry(const KernelDesc& kd, Index i, Index j);

}  // namespace midbf::ker
