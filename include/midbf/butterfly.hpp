// MIDBF factorize / apply — drop-in for the reference's
// proj/include/midbf/butterfly.hpp:24-135 (`midbf::bf`).
//
//   K ~ U^1 ... U^T  S  V^T ... V^1,  T = L - h + 1, h = ceil(L/2),
//
// stored as `factors = [U^1..U^T, S, V^T..V^1]` exactly as the reference
// (src/butterfly.cpp:765-767), so MIDBF001 files and block tables are
// interchangeable.  What changes is where the work runs:
//   * apply / apply_transpose run on the GPU (sm_100a kernels behind the
//     C ABI in include/midbf_b200.h); the host Factorization uploads itself
//     once into a device plan that is cached inside the object.
//   * idbf_factorize samples every kernel entry on the GPU when given a
//     `KernelDesc` (fused exp(2*pi*i*Phi) sampler); the EntryFn overload keeps
//     the reference's host-callback semantics for arbitrary kernels.
//   * with a `KernelDesc`, the interpolative decompositions run on the GPU
//     too (K5); the EntryFn overload runs them on the host (OpenMP).
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <utility>

#include "midbf/kernels.hpp"
#include "midbf/linalg.hpp"
#include "midbf/tree.hpp"
#include "midbf/types.hpp"

namespace midbf::bf {

using EntryFn = std::function<Cplx(Index, Index)>;  // :24

struct FactorBlock {  // :27-31
  Index row_off = 0;
  Index col_off = 0;
  MatXc M;
};

struct Factor {  // :37-45
  Index rows = 0;
  Index cols = 0;
  std::vector<FactorBlock> blocks;
  std::vector<std::pair<Index, Index>> groups;
  Index nnz() const;
};

struct Config {  // :46-51
  la::RankSpec rank{30, 1e-9};
  Index t = 5;
  std::uint64_t seed = 0;
  Exec exec = Exec::Serial;
};

struct DevicePlanCache;  // opaque: device arenas built from this object

// Holder of a Factorization's device-plan cache.  A copy starts empty (the
// copy builds its own plan on its first apply), so editing either object
// after a copy never reaches the other's arenas; moves keep the cache
// (the block buffers move with it).
struct DevicePlanSlot {
  std::shared_ptr<DevicePlanCache> p;
  DevicePlanSlot() = default;
  DevicePlanSlot(const DevicePlanSlot&) {}
  DevicePlanSlot& operator=(const DevicePlanSlot&) {
    p.reset();
    return *this;
  }
  DevicePlanSlot(DevicePlanSlot&&) noexcept = default;
  DevicePlanSlot& operator=(DevicePlanSlot&&) noexcept = default;
};

struct Factorization {  // :53-70
  Index nrows = 0;
  Index ncols = 0;
  int L = 0;
  int h = 0;
  Index n0 = 0;
  Config cfg;
  IndexVec row_perm;
  IndexVec col_perm;
  std::vector<Factor> factors;

  Index factor_count() const { return static_cast<Index>(factors.size()); }
  Index total_nnz() const;
  Index max_factor_nnz() const;
  double nnz_bound(double c = 4.0) const;

  // Device-plan cache (not part of the reference struct).  Built on the
  // first apply and rebuilt when the block layout changes (blocks added,
  // removed, reallocated or reshaped, perms resized); call
  // invalidate_device_plan() after editing block VALUES in place.  Thread
  // safe against concurrent applies (same lock as the cache lookup).
  mutable DevicePlanSlot device;
  void invalidate_device_plan() const;
};

// Reference overload: entries from a host callback (src/butterfly.cpp:708).
Factorization idbf_factorize(const EntryFn& K, const tree::ClusterTree& tx, const tree::ClusterTree& tomega,
                             const MatXd& X, const MatXd& Omega, const Config& cfg);

// B200 overload: every entry sampled on the GPU from a typed kernel
// description (explicit 2D/3D FIO phase, low-rank A*B^T phase, x.xi), and
// every ID computed there (K5; blocks the device hands back are redone on
// the host).
Factorization idbf_factorize(const ker::KernelDesc& K, const tree::ClusterTree& tx, const tree::ClusterTree& tomega,
                             const MatXd& X, const MatXd& Omega, const Config& cfg);

// g = F f and f = F^T g (plain transpose), on the GPU.  VecXc and MatXc are
// the same column-major type here, so one overload serves the reference's
// vector and multi-RHS forms (:123-126): f is N x nrhs, nrhs >= 1.  Throws
// std::invalid_argument on a length mismatch (src/butterfly.cpp:645) and
// std::runtime_error on a CUDA failure.
MatXc apply(const Factorization& F, const MatXc& fs);
MatXc apply_transpose(const Factorization& F, const MatXc& gs);

MatXc factor_dense(const Factor& F);
MatXc dense(const Factorization& F);

}  // namespace midbf::bf
