// Internal glue between the C++ host API and the C ABI.
#pragma once

#include <cstdint>
#include <memory>
#include <random>
#include <vector>

#include "midbf/butterfly.hpp"
#include "midbf_b200.h"

namespace midbf::la {

// mock_chebyshev_points in parts (linalg.cpp): the candidate search also runs
// on the GPU with the same arithmetic (dev::EntrySampler::cheb_candidates).
constexpr Index kChebCand = 8;  // nearest points kept per node, by (distance, index)
struct ChebNodes {
  Index c = 0, d = 0, nodes = 0;
  std::vector<double> nodec;  // nodes x d, row-major
};
ChebNodes cheb_nodes(const MatXd& P, Index s);
void cheb_candidates(const MatXd& P, const ChebNodes& N, Index* cand);  // nodes x kChebCand, -1: none
void cheb_candidates_node(const MatXd& P, const ChebNodes& N, Index t, Index* cand);  // node t's kChebCand
IndexVec cheb_pick(const MatXd& P, Index s, const ChebNodes& N, const Index* cand, std::mt19937_64& rng);

}  // namespace midbf::la

namespace midbf::bf {

struct FactorizeStats {
  std::int64_t entries = 0;   // kernel entries sampled on the device
  std::int64_t launches = 0;  // sampler calls (one per sweep pass)
  double sample_seconds = 0;  // wall time inside the device sampler (kernel + copies)
  std::int64_t device_ids = 0;    // IDs computed on the device (K5)
  std::int64_t id_fallbacks = 0;  // IDs the device handed back to the host
  double id_seconds = 0;          // wall time inside K3 + K5 ID batches (incl. copies)
  double seconds = 0;             // whole factorization
  // device time of the sampler's kernels (CUDA events): K3 entry sampling, K5 IDs
  std::int64_t k3_launches = 0, k3_entries = 0, k5_launches = 0;
  double k3_seconds = 0, k5_seconds = 0;
};

Factorization idbf_factorize_stats(const ker::KernelDesc& K, const tree::ClusterTree& tx,
                                   const tree::ClusterTree& to, const MatXd& X, const MatXd& Om, const Config& cfg,
                                   FactorizeStats* stats, bool device_id);

// Device plan cached inside the factorization; built (or rebuilt with the
// union of directions) on demand.
struct DevicePlanCache {
  midbf_plan_t plan = nullptr;
  unsigned directions = 0;
  std::uint64_t stamp = 0;  // layout_stamp of the factorization it was built from
  ~DevicePlanCache();
};
// Returns the cache entry (not just the handle) so that a concurrent caller
// rebuilding the cache with more directions cannot free a plan still in use.
std::shared_ptr<DevicePlanCache> device_plan(const Factorization& F, unsigned directions);

}  // namespace midbf::bf
