// Host interpolative decompositions (reference src/linalg.cpp:23-107,
// 249-295, 329-400).
//
// Difference from the reference, by design: the pivoted QR stops after
// min(m, n, k_max) Householder steps and never forms Q.  Step j only reads
// the results of steps < j, so the first k_max pivots and rows of R are the
// ones the full factorization computes; id_rank then sees the same leading
// diagonal.  The only way the truncated diagonal could select a different
// rank is a diagonal that falls below 1e-14*|R00| inside the first k_max
// steps and rises again later (id_rank's tail trim, src/linalg.cpp:252); in
// that case the full factorization is recomputed, so results never differ.
#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <stdexcept>

#include "midbf/linalg.hpp"
#include "midbf_internal.hpp"

namespace midbf::la {
namespace {

inline double nrm2(const Cplx& z) { return z.real() * z.real() + z.imag() * z.imag(); }
inline Cplx cmul(const Cplx& a, const Cplx& b) {
  return {a.real() * b.real() - a.imag() * b.imag(), a.real() * b.imag() + a.imag() * b.real()};
}
inline Cplx cmulc(const Cplx& a, const Cplx& b) {  // conj(a) * b
  return {a.real() * b.real() + a.imag() * b.imag(), a.real() * b.imag() - a.imag() * b.real()};
}

PivotedQR householder_qr(const MatXc& A0, Index steps_cap) {
  MatXc A = A0;
  const Index m = A.rows(), n = A.cols();
  Index steps = std::min(m, n);
  if (steps_cap >= 0) steps = std::min(steps, steps_cap);
  PivotedQR out;
  out.perm.resize(static_cast<size_t>(n));
  std::iota(out.perm.begin(), out.perm.end(), Index{0});
  std::vector<double> cur(static_cast<size_t>(n)), ref(static_cast<size_t>(n));
  for (Index j = 0; j < n; ++j) {
    const Cplx* c = &A(0, j);
    double s = 0.0;
    for (Index i = 0; i < m; ++i) s += nrm2(c[i]);
    cur[j] = ref[j] = s;
  }
  std::vector<Cplx> v(static_cast<size_t>(m)), bv(static_cast<size_t>(m));
  Index k = 0;
  for (; k < steps; ++k) {
    // pivot: largest remaining norm, lowest position on ties
    Index p = k;
    for (Index j = k + 1; j < n; ++j)
      if (cur[j] > cur[p]) p = j;
    if (p != k) {
      std::swap_ranges(&A(0, k), &A(0, k) + m, &A(0, p));
      std::swap(out.perm[k], out.perm[p]);
      std::swap(cur[k], cur[p]);
      std::swap(ref[k], ref[p]);
    }
    Cplx* col = &A(0, k);
    double xs = 0.0;
    for (Index i = k; i < m; ++i) xs += nrm2(col[i]);
    const double xn = std::sqrt(xs);
    if (xn == 0.0) break;
    const Cplx a0 = col[k];
    const double aa = std::sqrt(nrm2(a0));
    const Cplx ph = aa == 0.0 ? Cplx(1.0, 0.0) : a0 / aa;
    const Cplx v0 = a0 + ph * xn;
    for (Index i = k + 1; i < m; ++i) col[i] /= v0;
    double vs = 0.0;
    for (Index i = k + 1; i < m; ++i) vs += nrm2(col[i]);
    const double beta = 2.0 / (1.0 + vs);
    col[k] = -ph * xn;
    // H = I - beta v v^H on the trailing columns, v = [1; col(k+1:m)]
    const Index len = m - k;
    v[0] = Cplx(1.0, 0.0);
    for (Index i = 1; i < len; ++i) v[i] = col[k + i];
    for (Index i = 0; i < len; ++i) bv[i] = Cplx(beta * v[i].real(), beta * v[i].imag());
    for (Index j = k + 1; j < n; ++j) {
      Cplx* c = &A(k, j);
      Cplx w(0.0, 0.0);
      for (Index i = 0; i < len; ++i) w += cmulc(c[i], v[i]);
      const Cplx cw = std::conj(w);
      for (Index i = 0; i < len; ++i) c[i] -= cmul(bv[i], cw);
      // norm downdate with the reference's recompute guard
      cur[j] -= nrm2(c[0]);
      if (cur[j] < 0.0 || cur[j] <= 1e-12 * ref[j]) {
        double s = 0.0;
        for (Index i = 1; i < len; ++i) s += nrm2(c[i]);
        cur[j] = len > 1 ? s : 0.0;
        ref[j] = cur[j];
      }
    }
  }
  out.rank = k;
  out.R = MatXc(k, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i <= std::min(j, k - 1); ++i) out.R(i, j) = A(i, j);
  // unitary phase fix: real non-negative diagonal
  for (Index i = 0; i < k; ++i) {
    const double d = std::sqrt(nrm2(out.R(i, i)));
    if (d == 0.0) continue;
    const Cplx inv = Cplx(1.0, 0.0) / (out.R(i, i) / d);
    for (Index j = i; j < n; ++j) out.R(i, j) *= inv;
  }
  return out;
}

}  // namespace

PivotedQR pivoted_qr(const MatXc& A, Index max_steps) { return householder_qr(A, max_steps); }

Index id_rank(const VecXd& d, const RankSpec& spec) {
  Index m = d.size();
  if (m == 0 || d(0) == 0.0) return 0;
  while (m > 0 && d(m - 1) <= 1e-14 * d(0)) --m;
  Index k = m;
  if (spec.eps > 0.0)
    for (Index i = 0; i < m; ++i)
      if (d(i) <= spec.eps * d(0)) {
        k = i + 1;
        break;
      }
  if (spec.k_max > 0) k = std::min(k, spec.k_max);
  return k;
}

ColumnID cid_from_rows(const MatXc& B, const RankSpec& spec) {
  const Index m = B.rows(), n = B.cols();
  const Index full = std::min(m, n);
  Index cap = spec.k_max > 0 ? std::min(full, spec.k_max) : full;
  PivotedQR qr = householder_qr(B, cap);
  auto diag = [&](const PivotedQR& q) {
    VecXd d(q.rank, 1);
    for (Index i = 0; i < q.rank; ++i) d(i) = std::abs(q.R(i, i));
    return d;
  };
  VecXd d = diag(qr);
  if (qr.rank == cap && cap < full && qr.rank > 0) {
    bool tiny = false;
    for (Index i = 0; i < qr.rank; ++i) tiny = tiny || d(i) <= 1e-14 * d(0);
    if (tiny) {  // see the file comment: fall back to the full factorization
      qr = householder_qr(B, -1);
      d = diag(qr);
    }
  }
  const Index k = id_rank(d, spec);
  ColumnID out;
  out.rank = k;
  out.skeleton.assign(qr.perm.begin(), qr.perm.begin() + k);
  out.V = MatXc(k, n);
  // V(:, perm) = [I, R1^{-1} R2]; back substitution per trailing column
  std::vector<Cplx> x(static_cast<size_t>(k));
  for (Index j = 0; j < n; ++j) {
    if (j < k) {
      out.V(j, qr.perm[j]) = Cplx(1.0, 0.0);
      continue;
    }
    for (Index i = k - 1; i >= 0; --i) {
      Cplx s = qr.R(i, j);
      for (Index l = i + 1; l < k; ++l) s -= qr.R(i, l) * x[l];
      x[i] = s / qr.R(i, i);
    }
    for (Index i = 0; i < k; ++i) out.V(i, qr.perm[j]) = x[i];
  }
  return out;
}

RowID rid_from_cols(const MatXc& C, const RankSpec& spec) {
  MatXc Ct(C.cols(), C.rows());
  for (Index j = 0; j < C.cols(); ++j)
    for (Index i = 0; i < C.rows(); ++i) Ct(j, i) = C(i, j);
  ColumnID c = cid_from_rows(Ct, spec);
  RowID r;
  r.rank = c.rank;
  r.skeleton = std::move(c.skeleton);
  r.W = MatXc(C.rows(), r.rank);
  for (Index j = 0; j < c.V.cols(); ++j)
    for (Index i = 0; i < c.V.rows(); ++i) r.W(j, i) = c.V(i, j);
  return r;
}

// mock_chebyshev_points (src/linalg.cpp:329-388) in three parts, so that the
// candidate search (the O(n * c^d) part) can also run on the GPU
// (EntrySampler::cheb_candidates) with the same arithmetic:
//   cheb_nodes       c, the bounding box and the tensor nodes (last axis fastest);
//   cheb_candidates  each node's kChebCand nearest points by (distance, index);
//   cheb_pick        the picks in node order -- the first untaken candidate is
//                    the reference's "nearest unused point, first on ties"; a
//                    full scan when every candidate is taken -- then the random
//                    top-up and the sort.
ChebNodes cheb_nodes(const MatXd& P, Index s) {
  const Index n = P.rows(), d = P.cols();
  ChebNodes N;
  Index c = 1;  // largest c with c^d <= s
  while (std::pow(static_cast<double>(c + 1), static_cast<double>(d)) <= static_cast<double>(s)) ++c;
  std::vector<double> mid(static_cast<size_t>(d)), half(static_cast<size_t>(d));
  for (Index a = 0; a < d; ++a) {
    double lo = P(0, a), hi = P(0, a);
    for (Index i = 1; i < n; ++i) {
      lo = std::min(lo, P(i, a));
      hi = std::max(hi, P(i, a));
    }
    mid[a] = 0.5 * (lo + hi);
    half[a] = 0.5 * (hi - lo);
  }
  const double kPi = 3.14159265358979323846;
  Index nodes = 1;
  for (Index a = 0; a < d; ++a) nodes *= c;
  N.c = c;
  N.d = d;
  N.nodes = nodes;
  N.nodec.resize(static_cast<size_t>(nodes * d));
  for (Index t = 0; t < nodes; ++t) {
    Index rem = t;
    for (Index a = d - 1; a >= 0; --a) {
      const Index j = rem % c;
      rem /= c;
      N.nodec[static_cast<size_t>(t * d + a)] = mid[a] + half[a] * std::cos((2.0 * j + 1.0) * kPi / (2.0 * c));
    }
  }
  return N;
}

namespace {
double cheb_dist(const MatXd& P, const ChebNodes& N, Index i, Index t) {
  double dist = 0.0;
  for (Index a = 0; a < N.d; ++a) {
    const double e = P(i, a) - N.nodec[static_cast<size_t>(t * N.d + a)];
    dist += e * e;
  }
  return dist;
}
}  // namespace

void cheb_candidates_node(const MatXd& P, const ChebNodes& N, Index t, Index* ci) {
  const Index n = P.rows();
  double cd[kChebCand];
  for (Index q = 0; q < kChebCand; ++q) {
    cd[q] = std::numeric_limits<double>::infinity();
    ci[q] = -1;
  }
  for (Index i = 0; i < n; ++i) {
    const double dist = cheb_dist(P, N, i, t);
    if (!(dist < cd[kChebCand - 1])) continue;  // ties keep the earlier index
    Index q = kChebCand - 1;
    while (q > 0 && dist < cd[q - 1]) {
      cd[q] = cd[q - 1];
      ci[q] = ci[q - 1];
      --q;
    }
    cd[q] = dist;
    ci[q] = i;
  }
}

void cheb_candidates(const MatXd& P, const ChebNodes& N, Index* cand) {
#pragma omp parallel for schedule(dynamic) if (P.rows() * N.nodes >= (Index{1} << 20))
  for (Index t = 0; t < N.nodes; ++t) cheb_candidates_node(P, N, t, cand + t * kChebCand);
}

IndexVec cheb_pick(const MatXd& P, Index s, const ChebNodes& N, const Index* cand, std::mt19937_64& rng) {
  const Index n = P.rows(), nodes = N.nodes;
  std::vector<char> taken(static_cast<size_t>(n), 0);
  IndexVec picked;
  picked.reserve(static_cast<size_t>(s));
  for (Index t = 0; t < nodes; ++t) {
    Index best = -1;
    for (Index q = 0; q < kChebCand && best < 0; ++q) {
      const Index i = cand[static_cast<size_t>(t * kChebCand + q)];
      if (i >= 0 && !taken[i]) best = i;
    }
    if (best < 0) {  // all candidates taken: full scan over the untaken points
      double bd = std::numeric_limits<double>::infinity();
      for (Index i = 0; i < n; ++i) {
        if (taken[i]) continue;
        const double dist = cheb_dist(P, N, i, t);
        if (dist < bd) {
          bd = dist;
          best = i;
        }
      }
    }
    taken[best] = 1;
    picked.push_back(best);
  }
  IndexVec free_ids;
  for (Index i = 0; i < n; ++i)
    if (!taken[i]) free_ids.push_back(i);
  while (static_cast<Index>(picked.size()) < s && !free_ids.empty()) {
    std::uniform_int_distribution<size_t> pick(0, free_ids.size() - 1);
    const size_t at = pick(rng);
    picked.push_back(free_ids[at]);
    free_ids[at] = free_ids.back();
    free_ids.pop_back();
  }
  std::sort(picked.begin(), picked.end());
  return picked;
}

IndexVec mock_chebyshev_points(const MatXd& P, Index s, std::mt19937_64& rng) {
  const Index n = P.rows();
  IndexVec picked;
  if (s >= n) {
    picked.resize(static_cast<size_t>(n));
    std::iota(picked.begin(), picked.end(), Index{0});
    return picked;
  }
  const ChebNodes N = cheb_nodes(P, s);
  std::vector<Index> cand(static_cast<size_t>(N.nodes * kChebCand));
  cheb_candidates(P, N, cand.data());
  return cheb_pick(P, s, N, cand.data(), rng);
}

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

}  // namespace midbf::la
