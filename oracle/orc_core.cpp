// TEST INFRASTRUCTURE ONLY — CPU restatement ("oracle") of the reference
// MIDBF hot path.  Imported solely by tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs; never by the product.
//
// Parity status: the reference (proj/, C++20 + Eigen3 + OpenMP) cannot be
// compiled in this image (no Eigen headers, no gmpxx, no vendor/ doctest),
// so this file restates its algorithm and is pinned against the reference's
// own known-answer tests (tests/test_*.cpp pins ported in tests/).  Bitwise
// agreement with Eigen's internal summation orders is NOT claimed.
//
// Every function cites the reference file:line it follows
// (paths relative to /root/reference/proj).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <functional>
#include <limits>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "orc_core.hpp"

namespace orc {

// ---------------------------------------------------------------- RNG chain
// src/butterfly.cpp:20-27 (splitmix64 finalizer + chaining)
std::uint64_t mix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
std::uint64_t chain(std::uint64_t a, std::uint64_t b) { return mix64(a ^ mix64(b)); }

// ------------------------------------------------------------------ Morton
// src/geometry.cpp:15-33 (bit spreading) and :67-73 (first argument in the
// low bit of each digit).
static std::uint64_t spread2(std::uint64_t v) {
  v &= 0x1FFFFF;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFULL;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFULL;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0FULL;
  v = (v | (v << 2)) & 0x3333333333333333ULL;
  v = (v | (v << 1)) & 0x5555555555555555ULL;
  return v;
}
static std::uint64_t spread3(std::uint64_t v) {
  v &= 0x1FFFFF;
  v = (v | (v << 32)) & 0x001F00000000FFFFULL;
  v = (v | (v << 16)) & 0x001F0000FF0000FFULL;
  v = (v | (v << 8)) & 0x100F00F00F00F00FULL;
  v = (v | (v << 4)) & 0x10C30C30C30C30C3ULL;
  v = (v | (v << 2)) & 0x1249249249249249ULL;
  return v;
}

// ------------------------------------------------------------------- trees
// src/tree.cpp:16-26: 21-bit-per-axis key, coordinate 0 most significant.
static std::uint64_t cell_key(const double* t, int dim) {
  const int kBits = 21;
  std::uint32_t q[3] = {0, 0, 0};
  for (int a = 0; a < dim; ++a) {
    double s = std::floor(std::ldexp(t[a], kBits));
    if (s < 0.0) s = 0.0;
    const double top = std::ldexp(1.0, kBits) - 1;
    q[a] = static_cast<std::uint32_t>(s < top ? s : top);
  }
  if (dim == 3) return spread3(q[2]) | (spread3(q[1]) << 1) | (spread3(q[0]) << 2);
  return spread2(q[1]) | (spread2(q[0]) << 1);
}

// src/tree.cpp:30-114
Tree build_tree(const MatXd& X, Index n0, int min_depth) {
  const Index n = X.rows();
  const int dim = static_cast<int>(X.cols());
  if (n < 1) throw std::invalid_argument("build_tree: empty point set");
  if (dim != 2 && dim != 3) throw std::invalid_argument("build_tree: points must be 2D or 3D");
  if (n0 < 1) throw std::invalid_argument("build_tree: n0 must be positive");
  if (min_depth < 0 || min_depth > 21) throw std::invalid_argument("build_tree: min_depth out of range");

  double lo[3] = {0, 0, 0};
  double ext = 0.0;
  for (int a = 0; a < dim; ++a) {
    double mn = X(0, a), mx = X(0, a);
    for (Index i = 1; i < n; ++i) {
      mn = std::min(mn, X(i, a));
      mx = std::max(mx, X(i, a));
    }
    lo[a] = mn;
    ext = std::max(ext, mx - mn);
  }
  if (ext <= 0.0) ext = 1.0;

  std::vector<std::uint64_t> key(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) {
    double t[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a) t[a] = (X(i, a) - lo[a]) / ext;
    key[static_cast<size_t>(i)] = cell_key(t, dim);
  }

  Tree T;
  T.dim = dim;
  T.n0 = n0;
  T.perm.resize(static_cast<size_t>(n));
  std::iota(T.perm.begin(), T.perm.end(), Index{0});
  std::sort(T.perm.begin(), T.perm.end(), [&](Index a, Index b) {
    return key[a] != key[b] ? key[a] < key[b] : a < b;
  });
  const auto head = [&](Index pos, int level) {
    return key[static_cast<size_t>(T.perm[static_cast<size_t>(pos)])] >>
           (static_cast<unsigned>(21 - level) * static_cast<unsigned>(dim));
  };
  const auto widest = [&](int level) {
    Index w = 0;
    for (Index b = 0; b < n;) {
      Index e = b + 1;
      while (e < n && head(e, level) == head(b, level)) ++e;
      w = std::max(w, e - b);
      b = e;
    }
    return w;
  };
  int L = min_depth;
  while (L <= 21 && widest(L) > n0) ++L;
  if (L > 21) throw std::invalid_argument("build_tree: more than n0 points coincide at maximum refinement");
  T.depth = L;
  T.levels.resize(static_cast<size_t>(L + 1));
  for (int level = 0; level <= L; ++level) {
    auto& nodes = T.levels[static_cast<size_t>(level)];
    for (Index b = 0; b < n;) {
      Index e = b + 1;
      while (e < n && head(e, level) == head(b, level)) ++e;
      Node nd;
      nd.code = head(b, level);
      nd.begin = b;
      nd.end = e;
      nodes.push_back(nd);
      b = e;
    }
    if (level > 0) {
      auto& up = T.levels[static_cast<size_t>(level - 1)];
      Index p = 0;
      for (Index c = 0; c < static_cast<Index>(nodes.size()); ++c) {
        while (up[static_cast<size_t>(p)].code != (nodes[static_cast<size_t>(c)].code >> dim)) ++p;
        nodes[static_cast<size_t>(c)].parent = p;
        up[static_cast<size_t>(p)].child[nodes[static_cast<size_t>(c)].code & ((1u << dim) - 1)] = c;
        ++up[static_cast<size_t>(p)].nchild;
      }
    }
  }
  return T;
}

// ------------------------------------------------------------ pivoted QR
// src/linalg.cpp:23-107.  Householder with column pivoting (largest
// remaining norm, ties to the lowest position), norm downdating with the
// 1e-12 recompute guard, Q formed explicitly, diagonal phase-fixed to be
// real non-negative.
template <class S>
QR<S> pivoted_qr(Mat<S> A, Index max_rank) {
  const Index m = A.rows(), n = A.cols();
  Index steps = std::min(m, n);
  if (max_rank >= 0) steps = std::min(steps, max_rank);
  QR<S> out;
  out.perm.resize(static_cast<size_t>(n));
  std::iota(out.perm.begin(), out.perm.end(), Index{0});
  std::vector<double> nrm(static_cast<size_t>(n)), nrm0(static_cast<size_t>(n));
  for (Index j = 0; j < n; ++j) {
    double s = 0.0;
    for (Index i = 0; i < m; ++i) s += abs2(A(i, j));
    nrm[j] = nrm0[j] = s;
  }
  std::vector<S> tau(static_cast<size_t>(std::max<Index>(steps, 0)), S(0));
  Index done = 0;
  for (Index k = 0; k < steps; ++k) {
    Index p = k;
    for (Index j = k + 1; j < n; ++j)
      if (nrm[j] > nrm[p]) p = j;
    if (p != k) {
      for (Index i = 0; i < m; ++i) std::swap(A(i, k), A(i, p));
      std::swap(out.perm[k], out.perm[p]);
      std::swap(nrm[k], nrm[p]);
      std::swap(nrm0[k], nrm0[p]);
    }
    double xs = 0.0;
    for (Index i = k; i < m; ++i) xs += abs2(A(i, k));
    const double xn = std::sqrt(xs);
    if (xn == 0.0) break;
    const S a0 = A(k, k);
    const double aa = std::sqrt(abs2(a0));
    const S ph = (aa == 0.0) ? S(1) : S(a0 / aa);
    const S v0 = a0 + ph * xn;
    for (Index i = k + 1; i < m; ++i) A(i, k) /= v0;
    double vs = 0.0;
    for (Index i = k + 1; i < m; ++i) vs += abs2(A(i, k));
    tau[k] = S(2.0 / (1.0 + vs));
    A(k, k) = -ph * xn;
    if (k + 1 < n) {
      const Index len = m - k;
      std::vector<S> v(static_cast<size_t>(len));
      v[0] = S(1);
      for (Index i = 1; i < len; ++i) v[i] = A(k + i, k);
      std::vector<S> bv(static_cast<size_t>(len));
      for (Index i = 0; i < len; ++i) bv[i] = tau[k] * v[i];
      for (Index j = k + 1; j < n; ++j) {
        S w = S(0);
        for (Index i = 0; i < len; ++i) w += conj_(A(k + i, j)) * v[i];
        const S cw = conj_(w);
        for (Index i = 0; i < len; ++i) A(k + i, j) -= bv[i] * cw;
      }
    }
    for (Index j = k + 1; j < n; ++j) {
      nrm[j] -= abs2(A(k, j));
      if (nrm[j] < 0.0 || nrm[j] <= 1e-12 * nrm0[j]) {
        double s = 0.0;
        for (Index i = k + 1; i < m; ++i) s += abs2(A(i, j));
        nrm[j] = (m - k - 1 > 0) ? s : 0.0;
        nrm0[j] = nrm[j];
      }
    }
    done = k + 1;
  }
  out.rank = done;
  out.R = Mat<S>(done, n);
  for (Index i = 0; i < done; ++i)
    for (Index j = i; j < n; ++j) out.R(i, j) = A(i, j);
  out.Q = Mat<S>(m, done);
  for (Index i = 0; i < std::min(m, done); ++i) out.Q(i, i) = S(1);
  for (Index k = done - 1; k >= 0; --k) {
    const Index len = m - k;
    std::vector<S> v(static_cast<size_t>(len));
    v[0] = S(1);
    for (Index i = 1; i < len; ++i) v[i] = A(k + i, k);
    std::vector<S> bv(static_cast<size_t>(len));
    for (Index i = 0; i < len; ++i) bv[i] = tau[k] * v[i];
    for (Index j = k; j < done; ++j) {
      S w = S(0);
      for (Index i = 0; i < len; ++i) w += conj_(out.Q(k + i, j)) * v[i];
      const S cw = conj_(w);
      for (Index i = 0; i < len; ++i) out.Q(k + i, j) -= bv[i] * cw;
    }
  }
  for (Index k = 0; k < done; ++k) {
    const double dk = std::sqrt(abs2(out.R(k, k)));
    if (dk == 0.0) continue;
    const S ph = S(out.R(k, k) / dk);
    const S inv = S(1) / ph;
    for (Index j = 0; j < n; ++j) out.R(k, j) *= inv;
    for (Index i = 0; i < m; ++i) out.Q(i, k) *= ph;
  }
  return out;
}
template QR<double> pivoted_qr<double>(MatXd, Index);
template QR<Cplx> pivoted_qr<Cplx>(MatXc, Index);

// src/linalg.cpp:249-264
Index id_rank(const std::vector<double>& dg, Index k_max, double eps) {
  Index m = static_cast<Index>(dg.size());
  if (m == 0 || dg[0] == 0.0) return 0;
  while (m > 0 && dg[m - 1] <= 1e-14 * dg[0]) --m;
  Index k = m;
  if (eps > 0.0) {
    for (Index i = 0; i < m; ++i)
      if (dg[i] <= eps * dg[0]) {
        k = i + 1;
        break;
      }
  }
  if (k_max > 0) k = std::min(k, k_max);
  return k;
}

// src/linalg.cpp:266-286: V = [I, R1^{-1} R2] P^T from a full pivoted QR.
ColumnID cid_from_rows(const MatXc& blk, Index k_max, double eps) {
  const Index n = blk.cols();
  QR<Cplx> qr = pivoted_qr<Cplx>(blk, -1);
  std::vector<double> dg(static_cast<size_t>(qr.rank));
  for (Index i = 0; i < qr.rank; ++i) dg[i] = std::abs(qr.R(i, i));
  const Index k = id_rank(dg, k_max, eps);
  ColumnID out;
  out.rank = k;
  out.skeleton.assign(qr.perm.begin(), qr.perm.begin() + k);
  MatXc Vp(k, n);
  for (Index i = 0; i < k; ++i) Vp(i, i) = Cplx(1, 0);
  // Back substitution R1 * X = R2, one right-hand side column at a time.
  for (Index j = k; j < n; ++j) {
    for (Index i = k - 1; i >= 0; --i) {
      Cplx s = qr.R(i, j);
      for (Index l = i + 1; l < k; ++l) s -= qr.R(i, l) * Vp(l, j);
      Vp(i, j) = s / qr.R(i, i);
    }
  }
  out.V = MatXc(k, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < k; ++i) out.V(i, qr.perm[j]) = Vp(i, j);
  return out;
}

static MatXc transposed(const MatXc& A) {
  MatXc B(A.cols(), A.rows());
  for (Index j = 0; j < A.cols(); ++j)
    for (Index i = 0; i < A.rows(); ++i) B(j, i) = A(i, j);
  return B;
}

// src/linalg.cpp:288-295: plain-transpose dual of the column ID.
RowID rid_from_cols(const MatXc& blk, Index k_max, double eps) {
  ColumnID c = cid_from_rows(transposed(blk), k_max, eps);
  RowID r;
  r.skeleton = std::move(c.skeleton);
  r.W = transposed(c.V);
  r.rank = c.rank;
  return r;
}

// src/linalg.cpp:297-327
IndexVec mock_chebyshev_rows(const std::vector<double>& pts, Index s) {
  const Index n = static_cast<Index>(pts.size());
  if (s >= n) {
    IndexVec all(static_cast<size_t>(n));
    std::iota(all.begin(), all.end(), Index{0});
    return all;
  }
  double lo = pts[0], hi = pts[0];
  for (double v : pts) {
    lo = std::min(lo, v);
    hi = std::max(hi, v);
  }
  const double mid = 0.5 * (lo + hi), half = 0.5 * (hi - lo);
  const double kPi = 3.14159265358979323846;
  std::vector<char> used(static_cast<size_t>(n), 0);
  IndexVec got;
  for (Index j = 0; j < s; ++j) {
    const double node = mid + half * std::cos((2.0 * j + 1.0) * kPi / (2.0 * s));
    Index best = -1;
    double bd = std::numeric_limits<double>::infinity();
    for (Index i = 0; i < n; ++i) {
      if (used[i]) continue;
      const double dd = std::abs(pts[i] - node);
      if (dd < bd) {
        bd = dd;
        best = i;
      }
    }
    used[best] = 1;
    got.push_back(best);
  }
  std::sort(got.begin(), got.end());
  return got;
}

// src/linalg.cpp:329-388: tensor Chebyshev grid of c^d <= s nodes snapped to
// the nearest unused point (strict <, lowest index on ties), random top-up.
IndexVec mock_chebyshev_points(const MatXd& P, Index s, std::mt19937_64& rng) {
  const Index n = P.rows(), d = P.cols();
  if (s >= n) {
    IndexVec all(static_cast<size_t>(n));
    std::iota(all.begin(), all.end(), Index{0});
    return all;
  }
  Index c = 1;
  while (std::pow(static_cast<double>(c + 1), static_cast<double>(d)) <= static_cast<double>(s)) ++c;
  std::vector<double> lo(static_cast<size_t>(d)), hi(static_cast<size_t>(d));
  for (Index a = 0; a < d; ++a) {
    lo[a] = P(0, a);
    hi[a] = P(0, a);
    for (Index i = 1; i < n; ++i) {
      lo[a] = std::min(lo[a], P(i, a));
      hi[a] = std::max(hi[a], P(i, a));
    }
  }
  const double kPi = 3.14159265358979323846;
  Index total = 1;
  for (Index a = 0; a < d; ++a) total *= c;
  std::vector<char> used(static_cast<size_t>(n), 0);
  IndexVec got;
  std::vector<double> node(static_cast<size_t>(d));
  for (Index t = 0; t < total; ++t) {
    Index rem = t;
    for (Index a = d - 1; a >= 0; --a) {
      const Index j = rem % c;
      rem /= c;
      const double mid = 0.5 * (lo[a] + hi[a]), half = 0.5 * (hi[a] - lo[a]);
      node[a] = mid + half * std::cos((2.0 * j + 1.0) * kPi / (2.0 * c));
    }
    Index best = -1;
    double bd = std::numeric_limits<double>::infinity();
    for (Index i = 0; i < n; ++i) {
      if (used[i]) continue;
      double dist = 0.0;
      for (Index a = 0; a < d; ++a) {
        const double e = P(i, a) - node[a];
        dist += e * e;
      }
      if (dist < bd) {
        bd = dist;
        best = i;
      }
    }
    used[best] = 1;
    got.push_back(best);
  }
  IndexVec unused;
  for (Index i = 0; i < n; ++i)
    if (!used[i]) unused.push_back(i);
  while (static_cast<Index>(got.size()) < s && !unused.empty()) {
    std::uniform_int_distribution<size_t> pick(0, unused.size() - 1);
    const size_t pos = pick(rng);
    got.push_back(unused[pos]);
    unused[pos] = unused.back();
    unused.pop_back();
  }
  std::sort(got.begin(), got.end());
  return got;
}

// src/linalg.cpp:390-400
IndexVec rand_subset(Index n, Index k, std::mt19937_64& rng) {
  k = std::min(k, n);
  IndexVec pool(static_cast<size_t>(n));
  std::iota(pool.begin(), pool.end(), Index{0});
  for (Index i = 0; i < k; ++i) {
    std::uniform_int_distribution<Index> pick(i, n - 1);
    std::swap(pool[i], pool[pick(rng)]);
  }
  pool.resize(static_cast<size_t>(k));
  return pool;
}

// --------------------------------------------------- butterfly factorize
namespace {

struct Run {  // reference `Unit` (src/butterfly.cpp:31-35)
  Index node = 0;
  Index begin = 0;
  IndexVec ids;
};
struct Half {  // reference `Side` (src/butterfly.cpp:38-43)
  int level = 0;
  std::vector<Run> runs;
  Index size = 0;
  Index off = 0;
};
struct Sys {
  Half row, col;
};
struct Interp {  // reference `UnitID` (src/butterfly.cpp:347-350)
  MatXc M;
  IndexVec skel;
};
struct SweepResult {
  Factor U, V, S;
  Index mid_rows = 0, mid_cols = 0;
  std::vector<Sys> next;
};

Index up_to(const Tree& t, Index node, int from, int to) {  // :50-54
  for (int l = from; l > to; --l) node = t.levels[static_cast<size_t>(l)][static_cast<size_t>(node)].parent;
  return node;
}

Half leaves_of(const Tree& t) {  // :279-293
  Half h;
  h.level = t.depth;
  const auto& lv = t.levels[static_cast<size_t>(t.depth)];
  for (Index q = 0; q < static_cast<Index>(lv.size()); ++q) {
    Run r;
    r.node = q;
    r.begin = h.size;
    r.ids.assign(t.perm.begin() + lv[q].begin, t.perm.begin() + lv[q].end);
    h.size += static_cast<Index>(r.ids.size());
    h.runs.push_back(std::move(r));
  }
  return h;
}

// :360-369
IndexVec draw_ids(const IndexVec& pool, const MatXd& P, Index want, std::mt19937_64& rng) {
  const Index n = static_cast<Index>(pool.size());
  if (n <= want) return pool;
  MatXd C(n, P.cols());
  for (Index i = 0; i < n; ++i)
    for (Index a = 0; a < P.cols(); ++a) C(i, a) = P(pool[i], a);
  IndexVec sel = mock_chebyshev_points(C, want, rng);
  IndexVec out(sel.size());
  for (size_t i = 0; i < sel.size(); ++i) out[i] = pool[static_cast<size_t>(sel[i])];
  return out;
}

struct Frag {
  Index anc = -1;
  Half half;
};

// :380-408
std::vector<Frag> regroup(const Tree& tr, const Half& old, const std::vector<Interp>& ids, int level,
                          Index base) {
  std::vector<Frag> fr;
  Index used = 0;
  for (Index q = 0; q < static_cast<Index>(old.runs.size()); ++q) {
    const Run& r = old.runs[q];
    const Index anc = up_to(tr, r.node, old.level, level);
    if (fr.empty() || fr.back().anc != anc) {
      Frag f;
      f.anc = anc;
      f.half.level = old.level - 1;
      f.half.off = base + used;
      fr.push_back(std::move(f));
    }
    Half& nh = fr.back().half;
    const Index par = tr.levels[static_cast<size_t>(old.level)][static_cast<size_t>(r.node)].parent;
    if (nh.runs.empty() || nh.runs.back().node != par) {
      Run nr;
      nr.node = par;
      nr.begin = nh.size;
      nh.runs.push_back(std::move(nr));
    }
    const IndexVec& sk = ids[q].skel;
    nh.runs.back().ids.insert(nh.runs.back().ids.end(), sk.begin(), sk.end());
    nh.size += static_cast<Index>(sk.size());
    used += static_cast<Index>(sk.size());
  }
  return fr;
}

// :413-622
SweepResult sweep(const EntryFn& K, const Tree& tx, const Tree& to, const MatXd& X, const MatXd& Om,
                  const Config& cfg, const std::vector<Sys>& sys, Index nB, int level, bool last,
                  std::uint64_t salt, Index stage_rows, Index stage_cols) {
  const Index ns = static_cast<Index>(sys.size());
  const Index nA = ns / std::max<Index>(nB, 1);
  const Index want = cfg.k_max * cfg.t;
  const bool par = cfg.parallel;
  for (Index a = 0; a < nA; ++a)
    for (Index b = 1; b < nB; ++b)
      if (sys[a * nB + b].row.runs.size() != sys[a * nB].row.runs.size())
        throw std::logic_error("row unit layout differs between sibling systems");
  for (Index b = 0; b < nB; ++b)
    for (Index a = 1; a < nA; ++a)
      if (sys[a * nB + b].col.runs.size() != sys[b].col.runs.size())
        throw std::logic_error("column unit layout differs between sibling systems");

  std::vector<IndexVec> cs(static_cast<size_t>(ns));
  for (Index s = 0; s < ns; ++s) {
    IndexVec pool;
    for (const Run& w : sys[s].col.runs) pool.insert(pool.end(), w.ids.begin(), w.ids.end());
    std::mt19937_64 rng(chain(chain(salt, 0x73636f6cull), static_cast<std::uint64_t>(s)));
    cs[s] = draw_ids(pool, Om, want, rng);
  }

  std::vector<std::vector<Interp>> rid(static_cast<size_t>(ns));
  std::vector<std::pair<Index, Index>> rt;
  for (Index s = 0; s < ns; ++s) {
    rid[s].resize(sys[s].row.runs.size());
    for (Index u = 0; u < static_cast<Index>(sys[s].row.runs.size()); ++u) rt.emplace_back(s, u);
  }
#pragma omp parallel for schedule(dynamic) if (par)
  for (std::int64_t ti = 0; ti < static_cast<std::int64_t>(rt.size()); ++ti) {
    const Index s = rt[ti].first, u = rt[ti].second;
    const Run& r = sys[s].row.runs[u];
    const Index nu = static_cast<Index>(r.ids.size()), nc = static_cast<Index>(cs[s].size());
    Interp& o = rid[s][u];
    if (nu == 0 || nc == 0) {
      o.M = MatXc(nu, 0);
      continue;
    }
    MatXc blk(nu, nc);
    for (Index c = 0; c < nc; ++c)
      for (Index i = 0; i < nu; ++i) blk(i, c) = K(r.ids[i], cs[s][c]);
    RowID id = rid_from_cols(blk, cfg.k_max, cfg.eps);
    o.M = std::move(id.W);
    for (Index p : id.skeleton) o.skel.push_back(r.ids[p]);
  }

  std::vector<IndexVec> rhat(static_cast<size_t>(ns));
  std::vector<IndexVec> roff(static_cast<size_t>(ns));
  std::vector<Index> orow(static_cast<size_t>(ns), 0);
  Index mid_rows = 0;
  for (Index s = 0; s < ns; ++s) {
    orow[s] = mid_rows;
    roff[s].assign(rid[s].size(), 0);
    for (Index u = 0; u < static_cast<Index>(rid[s].size()); ++u) {
      roff[s][u] = static_cast<Index>(rhat[s].size());
      rhat[s].insert(rhat[s].end(), rid[s][u].skel.begin(), rid[s][u].skel.end());
    }
    mid_rows += static_cast<Index>(rhat[s].size());
  }

  std::vector<IndexVec> rs(static_cast<size_t>(ns));
  for (Index s = 0; s < ns; ++s) {
    std::mt19937_64 rng(chain(chain(salt, 0x73726f77ull), static_cast<std::uint64_t>(s)));
    rs[s] = draw_ids(rhat[s], X, want, rng);
  }

  std::vector<std::vector<Interp>> cid(static_cast<size_t>(ns));
  std::vector<std::pair<Index, Index>> ct;
  for (Index s = 0; s < ns; ++s) {
    cid[s].resize(sys[s].col.runs.size());
    for (Index w = 0; w < static_cast<Index>(sys[s].col.runs.size()); ++w) ct.emplace_back(s, w);
  }
#pragma omp parallel for schedule(dynamic) if (par)
  for (std::int64_t ti = 0; ti < static_cast<std::int64_t>(ct.size()); ++ti) {
    const Index s = ct[ti].first, w = ct[ti].second;
    const Run& r = sys[s].col.runs[w];
    const Index nw = static_cast<Index>(r.ids.size()), nr = static_cast<Index>(rs[s].size());
    Interp& o = cid[s][w];
    if (nw == 0 || nr == 0) {
      o.M = MatXc(0, nw);
      continue;
    }
    MatXc blk(nr, nw);
    for (Index c = 0; c < nw; ++c)
      for (Index i = 0; i < nr; ++i) blk(i, c) = K(rs[s][i], r.ids[c]);
    ColumnID id = cid_from_rows(blk, cfg.k_max, cfg.eps);
    o.M = std::move(id.V);
    for (Index p : id.skeleton) o.skel.push_back(r.ids[p]);
  }

  std::vector<IndexVec> chat(static_cast<size_t>(ns));
  std::vector<IndexVec> coff(static_cast<size_t>(ns));
  std::vector<Index> ocol(static_cast<size_t>(ns), 0);
  Index mid_cols = 0;
  for (Index s = 0; s < ns; ++s) {
    ocol[s] = mid_cols;
    coff[s].assign(cid[s].size(), 0);
    for (Index w = 0; w < static_cast<Index>(cid[s].size()); ++w) {
      coff[s][w] = static_cast<Index>(chat[s].size());
      chat[s].insert(chat[s].end(), cid[s][w].skel.begin(), cid[s][w].skel.end());
    }
    mid_cols += static_cast<Index>(chat[s].size());
  }

  SweepResult R;
  R.mid_rows = mid_rows;
  R.mid_cols = mid_cols;
  // U assembly (:539-563): blocks of sibling systems sharing output rows.
  R.U.rows = stage_rows;
  R.U.cols = mid_rows;
  for (Index a = 0; a < nA; ++a) {
    const Index nu = static_cast<Index>(sys[a * nB].row.runs.size());
    for (Index u = 0; u < nu; ++u) {
      Index g0 = static_cast<Index>(R.U.blocks.size());
      Index prev = -1;
      for (Index b = 0; b < nB; ++b) {
        const Index s = a * nB + b;
        MatXc& W = rid[s][u].M;
        if (W.rows() == 0 || W.cols() == 0) continue;
        const Index ro = sys[s].row.off + sys[s].row.runs[u].begin;
        if (prev >= 0 && ro != prev) {
          R.U.groups.emplace_back(g0, static_cast<Index>(R.U.blocks.size()));
          g0 = static_cast<Index>(R.U.blocks.size());
        }
        prev = ro;
        R.U.blocks.push_back({ro, orow[s] + roff[s][u], std::move(W)});
      }
      if (g0 < static_cast<Index>(R.U.blocks.size()))
        R.U.groups.emplace_back(g0, static_cast<Index>(R.U.blocks.size()));
    }
  }
  // V assembly (:565-588), mirrored over the column side.
  R.V.rows = mid_cols;
  R.V.cols = stage_cols;
  for (Index b = 0; b < nB; ++b) {
    const Index nw = static_cast<Index>(sys[b].col.runs.size());
    for (Index w = 0; w < nw; ++w) {
      Index g0 = static_cast<Index>(R.V.blocks.size());
      Index prev = -1;
      for (Index a = 0; a < nA; ++a) {
        const Index s = a * nB + b;
        MatXc& V = cid[s][w].M;
        if (V.rows() == 0 || V.cols() == 0) continue;
        const Index co = sys[s].col.off + sys[s].col.runs[w].begin;
        if (prev >= 0 && co != prev) {
          R.V.groups.emplace_back(g0, static_cast<Index>(R.V.blocks.size()));
          g0 = static_cast<Index>(R.V.blocks.size());
        }
        prev = co;
        R.V.blocks.push_back({ocol[s] + coff[s][w], co, std::move(V)});
      }
      if (g0 < static_cast<Index>(R.V.blocks.size()))
        R.V.groups.emplace_back(g0, static_cast<Index>(R.V.blocks.size()));
    }
  }
  if (last) {  // :590-604
    R.S.rows = mid_rows;
    R.S.cols = mid_cols;
    for (Index s = 0; s < ns; ++s) {
      const Index nr = static_cast<Index>(rhat[s].size()), nc = static_cast<Index>(chat[s].size());
      if (nr == 0 || nc == 0) continue;
      MatXc blk(nr, nc);
      for (Index c = 0; c < nc; ++c)
        for (Index i = 0; i < nr; ++i) blk(i, c) = K(rhat[s][i], chat[s][c]);
      const Index g = static_cast<Index>(R.S.blocks.size());
      R.S.blocks.push_back({orow[s], ocol[s], std::move(blk)});
      R.S.groups.emplace_back(g, g + 1);
    }
  } else {  // :605-620
    const Index na2 = static_cast<Index>(tx.levels[static_cast<size_t>(level)].size());
    const Index nb2 = static_cast<Index>(to.levels[static_cast<size_t>(level)].size());
    R.next.resize(static_cast<size_t>(na2 * nb2));
    for (Index s = 0; s < ns; ++s) {
      const auto rf = regroup(tx, sys[s].row, rid[s], level, orow[s]);
      const auto cf = regroup(to, sys[s].col, cid[s], level, ocol[s]);
      for (const Frag& a : rf)
        for (const Frag& b : cf) {
          Sys& nx = R.next[static_cast<size_t>(a.anc * nb2 + b.anc)];
          nx.row = a.half;
          nx.col = b.half;
        }
    }
  }
  return R;
}

Factor eye(Index n) {  // :329-335
  Factor f;
  f.rows = f.cols = n;
  MatXc I(n, n);
  for (Index i = 0; i < n; ++i) I(i, i) = Cplx(1, 0);
  f.blocks.push_back({0, 0, std::move(I)});
  f.groups.emplace_back(0, 1);
  return f;
}

}  // namespace

// :295-305 and :708-769
Factorization idbf_factorize(const EntryFn& K, const Tree& tx, const Tree& to, const MatXd& X,
                             const MatXd& Om, const Config& cfg) {
  if (tx.dim != to.dim) throw std::invalid_argument("row and column trees have different dimensions");
  if (X.rows() != static_cast<Index>(tx.perm.size()) || Om.rows() != static_cast<Index>(to.perm.size()))
    throw std::invalid_argument("point set sizes do not match the trees");
  if (X.cols() != tx.dim || Om.cols() != to.dim)
    throw std::invalid_argument("point coordinates do not match the tree dimension");
  if (cfg.k_max < 1) throw std::invalid_argument("rank cap must be positive");
  if (cfg.t < 1) throw std::invalid_argument("sampling oversize must be positive");
  if (tx.depth != to.depth) throw std::invalid_argument("butterfly factorization requires trees of equal depth");

  Factorization F;
  F.nrows = static_cast<Index>(tx.perm.size());
  F.ncols = static_cast<Index>(to.perm.size());
  F.L = tx.depth;
  F.h = (tx.depth + 1) / 2;
  F.n0 = tx.n0;
  F.cfg = cfg;
  F.row_perm = tx.perm;
  F.col_perm = to.perm;
  if (F.L == 0) {
    Factor S;
    S.rows = F.nrows;
    S.cols = F.ncols;
    MatXc Kd(F.nrows, F.ncols);
    for (Index c = 0; c < F.ncols; ++c)
      for (Index r = 0; r < F.nrows; ++r) Kd(r, c) = K(F.row_perm[r], F.col_perm[c]);
    S.blocks.push_back({0, 0, std::move(Kd)});
    S.groups.emplace_back(0, 1);
    F.factors.push_back(eye(F.nrows));
    F.factors.push_back(std::move(S));
    F.factors.push_back(eye(F.ncols));
    return F;
  }
  const int T = F.L - F.h + 1;
  std::vector<Sys> sys(1);
  sys[0].row = leaves_of(tx);
  sys[0].col = leaves_of(to);
  Index nB = 1, sr = F.nrows, sc = F.ncols;
  std::vector<Factor> Us, Vs;
  Factor S;
  for (int t = 1; t <= T; ++t) {
    SweepResult o = sweep(K, tx, to, X, Om, cfg, sys, nB, t, t == T, chain(cfg.seed, static_cast<std::uint64_t>(t)),
                          sr, sc);
    Us.push_back(std::move(o.U));
    Vs.push_back(std::move(o.V));
    if (t == T) {
      S = std::move(o.S);
    } else {
      sys = std::move(o.next);
      nB = static_cast<Index>(to.levels[static_cast<size_t>(t)].size());
      sr = o.mid_rows;
      sc = o.mid_cols;
    }
  }
  for (Factor& f : Us) F.factors.push_back(std::move(f));
  F.factors.push_back(std::move(S));
  for (auto it = Vs.rbegin(); it != Vs.rend(); ++it) F.factors.push_back(std::move(*it));
  return F;
}

// ------------------------------------------------------------------ apply
// src/butterfly.cpp:624-640: y = 0; per group (OpenMP dynamic), blocks in
// fixed order: y[rows] += M * x[cols] (or M^T for the transpose).
// Vectors are column-major (len x nrhs), complex interleaved.
static void factor_apply(const Factor& F, const std::vector<Cplx>& x, Index xlen, std::vector<Cplx>& y,
                         Index nrhs, bool tr, bool par) {
  const Index ylen = tr ? F.cols : F.rows;
  y.assign(static_cast<size_t>(ylen * nrhs), Cplx(0, 0));
  const std::int64_t ng = static_cast<std::int64_t>(F.groups.size());
#pragma omp parallel for schedule(dynamic) if (par)
  for (std::int64_t g = 0; g < ng; ++g) {
    for (Index bi = F.groups[g].first; bi < F.groups[g].second; ++bi) {
      const Block& b = F.blocks[bi];
      const Index m = b.M.rows(), n = b.M.cols();
      for (Index q = 0; q < nrhs; ++q) {
        if (!tr) {
          double* yo = reinterpret_cast<double*>(y.data() + q * ylen + b.row_off);
          const double* xi = reinterpret_cast<const double*>(x.data() + q * xlen + b.col_off);
          for (Index c = 0; c < n; ++c) {
            const double xr = xi[2 * c], xim = xi[2 * c + 1];
            const double* mc = reinterpret_cast<const double*>(b.M.col(c));
            for (Index i = 0; i < m; ++i) {
              yo[2 * i] += mc[2 * i] * xr - mc[2 * i + 1] * xim;
              yo[2 * i + 1] += mc[2 * i] * xim + mc[2 * i + 1] * xr;
            }
          }
        } else {
          double* yo = reinterpret_cast<double*>(y.data() + q * ylen + b.col_off);
          const double* xi = reinterpret_cast<const double*>(x.data() + q * xlen + b.row_off);
          for (Index c = 0; c < n; ++c) {
            const double* mc = reinterpret_cast<const double*>(b.M.col(c));
            double sr = 0.0, si = 0.0;
            for (Index i = 0; i < m; ++i) {
              sr += mc[2 * i] * xi[2 * i] - mc[2 * i + 1] * xi[2 * i + 1];
              si += mc[2 * i] * xi[2 * i + 1] + mc[2 * i + 1] * xi[2 * i];
            }
            yo[2 * c] += sr;
            yo[2 * c + 1] += si;
          }
        }
      }
    }
  }
}

// src/butterfly.cpp:642-667
void apply(const Factorization& F, const Cplx* in, Index nrhs, bool tr, Cplx* out, bool par) {
  const Index nin = tr ? F.nrows : F.ncols;
  const Index nout = tr ? F.ncols : F.nrows;
  const IndexVec& ip = tr ? F.row_perm : F.col_perm;
  const IndexVec& op = tr ? F.col_perm : F.row_perm;
  std::vector<Cplx> v(static_cast<size_t>(nin * nrhs)), w;
  for (Index q = 0; q < nrhs; ++q)
    for (Index p = 0; p < nin; ++p) v[q * nin + p] = in[q * nin + ip[p]];
  Index vlen = nin;
  const Index nf = static_cast<Index>(F.factors.size());
  for (Index s = 0; s < nf; ++s) {
    const Factor& fac = F.factors[tr ? s : nf - 1 - s];
    factor_apply(fac, v, vlen, w, nrhs, tr, par);
    vlen = tr ? fac.cols : fac.rows;
    v.swap(w);
  }
  for (Index q = 0; q < nrhs; ++q)
    for (Index p = 0; p < nout; ++p) out[q * nout + op[p]] = v[q * vlen + p];
}

Index Factorization::total_nnz() const {  // :671-681
  Index n = 0;
  for (const Factor& f : factors)
    for (const Block& b : f.blocks) n += b.M.size();
  return n;
}
Index Factorization::max_factor_nnz() const {  // :683-687
  Index best = 0;
  for (const Factor& f : factors) {
    Index n = 0;
    for (const Block& b : f.blocks) n += b.M.size();
    best = std::max(best, n);
  }
  return best;
}
double Factorization::nnz_bound(double c) const {  // :689-693
  const double k = static_cast<double>(cfg.k_max);
  const double N = static_cast<double>(std::max(nrows, ncols));
  return c * k * k / static_cast<double>(std::max<Index>(n0, 1)) * N;
}

// ------------------------------------------------------- MIDBF001 container
// src/butterfly_io.cpp:63-167 (layout documented at include/midbf/butterfly_io.hpp:2-15)
void save(const std::string& path, const Factorization& F) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open for writing: " + path);
  const auto i64 = [&](std::int64_t v) { f.write(reinterpret_cast<const char*>(&v), 8); };
  f.write("MIDBF001", 8);
  i64(F.nrows);
  i64(F.ncols);
  i64(F.L);
  i64(F.h);
  i64(F.n0);
  i64(F.cfg.k_max);
  i64(F.cfg.t);
  f.write(reinterpret_cast<const char*>(&F.cfg.eps), 8);
  const std::uint64_t seed = F.cfg.seed, ex = F.cfg.parallel ? 1 : 0;
  f.write(reinterpret_cast<const char*>(&seed), 8);
  f.write(reinterpret_cast<const char*>(&ex), 8);
  i64(static_cast<std::int64_t>(F.factors.size()));
  for (Index p : F.row_perm) i64(p);
  for (Index p : F.col_perm) i64(p);
  for (const Factor& fc : F.factors) {
    i64(fc.rows);
    i64(fc.cols);
    i64(static_cast<std::int64_t>(fc.blocks.size()));
    i64(static_cast<std::int64_t>(fc.groups.size()));
    for (const Block& b : fc.blocks) {
      i64(b.row_off);
      i64(b.col_off);
      i64(b.M.rows());
      i64(b.M.cols());
    }
    for (const auto& g : fc.groups) {
      i64(g.first);
      i64(g.second);
    }
  }
  for (const Factor& fc : F.factors)
    for (const Block& b : fc.blocks)
      f.write(reinterpret_cast<const char*>(b.M.d.data()), static_cast<std::streamsize>(16 * b.M.size()));
  if (!f) throw std::runtime_error("short write to " + path);
}

Factorization load(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open for reading: " + path);
  const auto need = [&](bool ok, const char* what) {
    if (!ok) throw std::runtime_error(std::string(what) + " in " + path);
  };
  const auto raw = [&]() {
    std::int64_t v = 0;
    f.read(reinterpret_cast<char*>(&v), 8);
    need(bool(f), "truncated container");
    return v;
  };
  const auto count = [&](const char* what, std::int64_t mx) {
    const std::int64_t v = raw();
    need(v >= 0 && v <= mx, what);
    return static_cast<Index>(v);
  };
  const std::int64_t big = std::int64_t{1} << 40;
  char magic[8];
  f.read(magic, 8);
  need(bool(f), "truncated container");
  need(std::memcmp(magic, "MIDBF001", 8) == 0, "unrecognized container magic");
  Factorization F;
  F.nrows = count("bad row count", big);
  F.ncols = count("bad column count", big);
  F.L = static_cast<int>(count("bad level count", 64));
  F.h = static_cast<int>(count("bad stop level", 64));
  F.n0 = count("bad leaf size", big);
  F.cfg.k_max = count("bad rank cap", big);
  F.cfg.t = count("bad sampling oversize", big);
  std::int64_t e = raw();
  std::memcpy(&F.cfg.eps, &e, 8);
  F.cfg.seed = static_cast<std::uint64_t>(raw());
  F.cfg.parallel = raw() != 0;
  const Index nf = count("bad factor count", 4096);
  F.row_perm.resize(static_cast<size_t>(F.nrows));
  for (Index i = 0; i < F.nrows; ++i) {
    F.row_perm[i] = count("bad row permutation entry", big);
    need(F.row_perm[i] < F.nrows, "row permutation out of range");
  }
  F.col_perm.resize(static_cast<size_t>(F.ncols));
  for (Index i = 0; i < F.ncols; ++i) {
    F.col_perm[i] = count("bad column permutation entry", big);
    need(F.col_perm[i] < F.ncols, "column permutation out of range");
  }
  F.factors.resize(static_cast<size_t>(nf));
  for (Factor& fc : F.factors) {
    fc.rows = count("bad factor rows", big);
    fc.cols = count("bad factor cols", big);
    const Index nb = count("bad block count", big), ng = count("bad group count", big);
    fc.blocks.resize(static_cast<size_t>(nb));
    for (Block& b : fc.blocks) {
      b.row_off = count("bad block row offset", big);
      b.col_off = count("bad block column offset", big);
      const Index m = count("bad block height", big), n = count("bad block width", big);
      need(b.row_off + m <= fc.rows && b.col_off + n <= fc.cols, "block outside its factor");
      b.M = MatXc(m, n);
    }
    fc.groups.resize(static_cast<size_t>(ng));
    for (auto& g : fc.groups) {
      g.first = count("bad group begin", big);
      g.second = count("bad group end", big);
      need(g.first <= g.second && g.second <= nb, "group outside block table");
    }
  }
  for (Factor& fc : F.factors)
    for (Block& b : fc.blocks) {
      f.read(reinterpret_cast<char*>(b.M.d.data()), static_cast<std::streamsize>(16 * b.M.size()));
      need(bool(f), "truncated payload");
    }
  f.peek();
  need(f.eof(), "trailing bytes after payload");
  return F;
}

// ----------------------------------------------------------------- kernels
namespace {
const double kTwoPi = 6.283185307179586476925286766559;
}

// src/kernels.cpp:18-24
double fio2d_phase(const double* x, const double* xi) {
  const double c1 = (2.0 + std::sin(kTwoPi * x[0]) * std::sin(kTwoPi * x[1])) / 16.0;
  const double c2 = (2.0 + std::cos(kTwoPi * x[0]) * std::cos(kTwoPi * x[1])) / 16.0;
  return x[0] * xi[0] + x[1] * xi[1] + std::sqrt(c1 * c1 * xi[0] * xi[0] + c2 * c2 * xi[1] * xi[1]);
}

// BASELINE.json configs[3] (not in the reference; its 2D formula extended).
double fio3d_phase(const double* x, const double* xi) {
  const double s0 = std::sin(kTwoPi * x[0]), s1 = std::sin(kTwoPi * x[1]), s2 = std::sin(kTwoPi * x[2]);
  const double c0 = std::cos(kTwoPi * x[0]), c1 = std::cos(kTwoPi * x[1]), c2 = std::cos(kTwoPi * x[2]);
  const double a1 = (2.0 + s0 * s1 * s2) / 16.0;
  const double a2 = (2.0 + c0 * c1 * c2) / 16.0;
  const double a3 = (2.0 + s0 * c1 * s2) / 16.0;
  return x[0] * xi[0] + x[1] * xi[1] + x[2] * xi[2] +
         std::sqrt(a1 * a1 * xi[0] * xi[0] + a2 * a2 * xi[1] * xi[1] + a3 * a3 * xi[2] * xi[2]);
}

// Entry function from a plain kernel description; mirrors make_accessor's
// scenario-1 entry polar(1, 2*pi*Phi) (src/kernels.cpp:242-245) and
// phase_entry_fn (src/metrics.cpp:18-24).  Point arrays are row-major N x dim.
EntryFn make_entry(const KernelDesc& kd) {
  switch (kd.kind) {
    case KIND_FIO2D:
      return [kd](Index i, Index j) {
        return std::polar(1.0, kTwoPi * fio2d_phase(kd.X + 2 * i, kd.Omega + 2 * j));
      };
    case KIND_FIO3D:
      return [kd](Index i, Index j) {
        return std::polar(1.0, kTwoPi * fio3d_phase(kd.X + 3 * i, kd.Omega + 3 * j));
      };
    case KIND_LOWRANK:
      return [kd](Index i, Index j) {
        double s = 0.0;
        for (int q = 0; q < kd.rank; ++q) s += kd.A[i * kd.rank + q] * kd.B[j * kd.rank + q];
        return std::polar(1.0, kTwoPi * s);
      };
    case KIND_NUFFT:
      return [kd](Index i, Index j) {
        double s = 0.0;
        for (int q = 0; q < kd.dim; ++q) s += kd.X[i * kd.dim + q] * kd.Omega[j * kd.dim + q];
        return std::polar(1.0, kTwoPi * s);
      };
    case KIND_CONST:
      return [kd](Index, Index) { return Cplx(kd.cre, kd.cim); };
    case KIND_RANK1:
      return [kd](Index i, Index j) {
        return Cplx(kd.u[2 * i], kd.u[2 * i + 1]) * Cplx(kd.v[2 * j], kd.v[2 * j + 1]);
      };
    default:
      throw std::invalid_argument("unknown kernel kind");
  }
}

// src/metrics.cpp:26-48 inner loop / tests/test_butterfly.cpp:29-37:
// g(i) = sum_j K(i,j) f(j) over the listed rows.
void direct_sum(const EntryFn& K, Index ncols, const Cplx* f, const Index* rows, Index nrows, Cplx* out,
                bool par) {
#pragma omp parallel for schedule(dynamic) if (par)
  for (std::int64_t q = 0; q < nrows; ++q) {
    Cplx acc(0, 0);
    for (Index j = 0; j < ncols; ++j) acc += K(rows[q], j) * f[j];
    out[q] = acc;
  }
}

// src/metrics.cpp:26-48
double eps_b_of(const Cplx* gb, Index N, const EntryFn& K, const Cplx* f, Index n, Index nrows,
                std::uint64_t seed) {
  if (nrows < 1) throw std::invalid_argument("eps_b: need at least one sampled row");
  std::mt19937_64 rng(seed);
  IndexVec S;
  if (nrows >= N) {
    S.resize(static_cast<size_t>(N));
    std::iota(S.begin(), S.end(), Index{0});
  } else {
    S = rand_subset(N, nrows, rng);
  }
  double num = 0.0, den = 0.0;
  for (Index i : S) {
    Cplx gd(0.0, 0.0);
    for (Index j = 0; j < n; ++j) gd += K(i, j) * f[j];
    num += std::norm(gb[i] - gd);
    den += std::norm(gd);
  }
  if (den == 0.0) return std::sqrt(num);
  return std::sqrt(num / den);
}

// src/experiment.cpp:75-81 — the same expression (argument evaluation order
// is compiler-defined; this file is built with the same g++ as the reference
// would be in this image).
void random_coefficients(Index n, std::uint64_t seed, Cplx* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> g(0.0, 1.0);
  for (Index i = 0; i < n; ++i) out[i] = Cplx(g(rng), g(rng));
}

// src/kernels.cpp:37-45 (row-major n*n x 2 here)
void grid2d(Index n, double* X) {
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < n; ++j) {
      X[2 * (i * n + j)] = double(i) / double(n);
      X[2 * (i * n + j) + 1] = double(j) / double(n);
    }
}

}  // namespace orc
