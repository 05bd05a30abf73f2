// Cluster trees (reference src/tree.cpp:16-114 and the Morton helpers of
// src/geometry.cpp:15-33, 67-73).  One 63-bit Morton key per point with 21
// bits per axis, the first coordinate in the most significant bit of each
// level digit; the depth is the smallest level >= min_depth whose occupied
// cells hold <= n0 points; every level lists its occupied cells in Morton
// order with contiguous ranges into `perm`.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>

#include "midbf/tree.hpp"

namespace midbf::tree {
namespace {

constexpr int kLevels = 21;

// Bit b of a 21-bit value moved to bit 2b (spread2) or 3b (spread3).
std::uint64_t spread2(std::uint64_t v) {
  v &= 0x1fffffull;
  v = (v | (v << 16)) & 0x0000ffff0000ffffull;
  v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
  v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}
std::uint64_t spread3(std::uint64_t v) {
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x001f00000000ffffull;
  v = (v | (v << 16)) & 0x001f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
// Interleave `dim` 21-bit coordinates; axis a lands at bit offset dim-1-a of
// every digit (axis 0 most significant).
std::uint64_t interleave(const std::uint32_t* q, int dim) {
  if (dim == 2) return (spread2(q[0]) << 1) | spread2(q[1]);
  return (spread3(q[0]) << 2) | (spread3(q[1]) << 1) | spread3(q[2]);
}

}  // namespace

ClusterTree build_tree(const MatXd& X, Index n0, int min_depth) {
  const Index n = X.rows();
  const int dim = static_cast<int>(X.cols());
  if (n < 1) throw std::invalid_argument("build_tree: empty point set");
  if (dim != 2 && dim != 3) throw std::invalid_argument("build_tree: points must be 2D or 3D");
  if (n0 < 1) throw std::invalid_argument("build_tree: n0 must be positive");
  if (min_depth < 0 || min_depth > kLevels) throw std::invalid_argument("build_tree: min_depth out of range");

  // Normalise by the largest bounding-box extent so cells stay square.
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  for (int a = 0; a < dim; ++a) {
    lo[a] = hi[a] = X(0, a);
    for (Index i = 1; i < n; ++i) {
      lo[a] = std::min(lo[a], X(i, a));
      hi[a] = std::max(hi[a], X(i, a));
    }
  }
  double ext = 0.0;
  for (int a = 0; a < dim; ++a) ext = std::max(ext, hi[a] - lo[a]);
  if (ext <= 0.0) ext = 1.0;
  const double scale = std::ldexp(1.0, kLevels), top = scale - 1.0;
  std::vector<std::uint64_t> key(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) {
    std::uint32_t q[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a) {
      // (x - lo) / ext * 2^21: scaling by a power of two is exact, as ldexp
      const double s = std::floor((X(i, a) - lo[a]) / ext * scale);
      q[a] = static_cast<std::uint32_t>(std::min(std::max(s, 0.0), top));
    }
    key[static_cast<size_t>(i)] = interleave(q, dim);
  }

  ClusterTree T;
  T.dim = dim;
  T.n0 = n0;
  T.perm.resize(static_cast<size_t>(n));
  {  // stable order by key: LSD radix sort, 8 bits per pass over the key's 21*dim bits
    std::vector<Index> tmp(static_cast<size_t>(n));
    std::iota(T.perm.begin(), T.perm.end(), Index{0});
    const int bits = kLevels * dim;
    for (int sh = 0; sh < bits; sh += 8) {
      size_t cnt[257] = {0};
      for (Index i = 0; i < n; ++i) ++cnt[((key[static_cast<size_t>(i)] >> sh) & 0xffu) + 1];
      for (int b = 0; b < 256; ++b) cnt[b + 1] += cnt[b];
      for (Index p = 0; p < n; ++p) {
        const Index i = T.perm[static_cast<size_t>(p)];
        tmp[cnt[(key[static_cast<size_t>(i)] >> sh) & 0xffu]++] = i;
      }
      T.perm.swap(tmp);
    }
  }
  T.pos_of.resize(static_cast<size_t>(n));
  for (Index p = 0; p < n; ++p) T.pos_of[static_cast<size_t>(T.perm[p])] = p;

  std::vector<std::uint64_t> sk(static_cast<size_t>(n));
  for (Index p = 0; p < n; ++p) sk[static_cast<size_t>(p)] = key[static_cast<size_t>(T.perm[p])];
  const auto cell = [&](Index p, int level) { return sk[static_cast<size_t>(p)] >> ((kLevels - level) * dim); };
  // Largest run of equal level-`level` prefixes in Morton order.
  const auto fullest = [&](int level) {
    Index best = 0, run = 1;
    for (Index p = 1; p <= n; ++p) {
      if (p < n && cell(p, level) == cell(p - 1, level)) {
        ++run;
      } else {
        best = std::max(best, run);
        run = 1;
      }
    }
    return best;
  };
  int L = min_depth;
  while (L <= kLevels && fullest(L) > n0) ++L;
  if (L > kLevels) throw std::invalid_argument("build_tree: more than n0 points coincide at maximum refinement");
  T.depth = L;
  T.levels.assign(static_cast<size_t>(L + 1), {});
  for (int level = 0; level <= L; ++level) {
    auto& nodes = T.levels[static_cast<size_t>(level)];
    Index start = 0;
    for (Index p = 1; p <= n; ++p) {
      if (p < n && cell(p, level) == cell(start, level)) continue;
      TreeNode nd;
      nd.code = cell(start, level);
      nd.begin = start;
      nd.end = p;
      if (level > 0) {
        auto& up = T.levels[static_cast<size_t>(level - 1)];
        // parents are in Morton order too: the parent of this run is the
        // last parent whose range starts at or before `start`.
        auto it = std::upper_bound(up.begin(), up.end(), start,
                                   [](Index v, const TreeNode& u) { return v < u.begin; });
        const Index par = static_cast<Index>(it - up.begin()) - 1;
        nd.parent = par;
        up[static_cast<size_t>(par)].child[nd.code & ((1u << dim) - 1)] = static_cast<Index>(nodes.size());
        ++up[static_cast<size_t>(par)].nchild;
      }
      nodes.push_back(nd);
      start = p;
    }
  }
  return T;
}

}  // namespace midbf::tree
