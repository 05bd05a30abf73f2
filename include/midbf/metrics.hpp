// Accuracy metrics against direct summation — drop-in for eps_b / eps_b_of of
// the reference's proj/include/midbf/metrics.hpp:15-28.  The direct sum runs
// on the GPU (midbf_direct_sum); the sampled-row selection follows the
// reference (rand_subset with std::mt19937_64(seed), src/metrics.cpp:30-38).
#pragma once

#include <cstdint>

#include "midbf/butterfly.hpp"
#include "midbf/kernels.hpp"

namespace midbf::metrics {

double eps_b(const bf::Factorization& F, const ker::KernelDesc& K, const VecXc& f, Index nrows, std::uint64_t seed);
double eps_b_of(const VecXc& g_b, const ker::KernelDesc& K, const VecXc& f, Index nrows, std::uint64_t seed);

}  // namespace midbf::metrics
