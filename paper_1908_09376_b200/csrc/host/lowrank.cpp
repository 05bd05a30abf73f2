// Low-rank phase production; see include/midbf/lowrank.hpp.
//
// la::rsvd restates src/linalg.cpp:134-219 step by step: pivoted QR of the
// sampled row slab (skeleton columns) and of the adjoint of the sampled
// column slab (skeleton rows), thin Q of the skeleton columns / rows,
// enlarged index sets (skeletons + rand_subset draws of the same sizes from
// `rng`), M = pinv(Qc(I,:)) A(I,J) pinv(Qr(J,:)^H), SVD of M, rank-r
// truncation.  Rows/columns are cached and counted as the reference does.
// The dense helpers differ from Eigen only where results are defined up to
// a unitary: thin_q is a Householder QR (basis phases may differ), and the
// SVDs are one-sided Jacobi (singular vectors defined up to phase; U S V^H,
// pinv and the singular values are the same up to rounding).
#include "midbf/lowrank.hpp"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <unordered_map>

#include "../device/sample.hpp"
#include "midbf/linalg.hpp"

namespace midbf::la {
namespace {

inline double abs2(double x) { return x * x; }
inline double abs2(const Cplx& x) { return x.real() * x.real() + x.imag() * x.imag(); }
inline double conj(double x) { return x; }
inline Cplx conj(const Cplx& x) { return std::conj(x); }

template <typename S>
Matrix<S> adjoint(const Matrix<S>& A) {
  Matrix<S> B(A.cols(), A.rows());
  for (Index j = 0; j < A.cols(); ++j)
    for (Index i = 0; i < A.rows(); ++i) B(j, i) = conj(A(i, j));
  return B;
}

template <typename S>
Matrix<S> matmul(const Matrix<S>& A, const Matrix<S>& B) {
  if (A.cols() != B.rows()) throw std::invalid_argument("matmul: inner dimensions differ");
  Matrix<S> C(A.rows(), B.cols());
  for (Index j = 0; j < B.cols(); ++j)
    for (Index l = 0; l < A.cols(); ++l) {
      const S b = B(l, j);
      if (b == S(0)) continue;
      for (Index i = 0; i < A.rows(); ++i) C(i, j) += A(i, l) * b;
    }
  return C;
}

// One-sided Jacobi (Hestenes) on m >= n: rotate column pairs of U = A until
// mutually orthogonal; V accumulates the rotations.  Complex pairs are first
// rephased so that u_p^H u_q is real.  Pairs follow a round-robin tournament
// (n-1 rounds of disjoint pairs), each round in parallel.
template <typename S>
bool rotate_pair(Matrix<S>& U, Matrix<S>& V, Index p, Index q, double tol) {
  const Index m = U.rows(), n = V.rows();
  double a = 0.0, b = 0.0;
  S g = S(0);
  for (Index i = 0; i < m; ++i) {
    a += abs2(U(i, p));
    b += abs2(U(i, q));
    g += conj(U(i, p)) * U(i, q);
  }
  const double ga = std::abs(g);
  if (ga == 0.0 || ga <= tol * std::sqrt(a * b)) return false;
  const S e = g / ga;  // phase of g; u_q <- u_q conj(e) makes the pair real
  const double zeta = (b - a) / (2.0 * ga);
  const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
  const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
  const S ec = conj(e);
  for (Index i = 0; i < m; ++i) {
    const S up = U(i, p), uq = U(i, q) * ec;
    U(i, p) = c * up - sn * uq;
    U(i, q) = sn * up + c * uq;
  }
  for (Index i = 0; i < n; ++i) {
    const S vp = V(i, p), vq = V(i, q) * ec;
    V(i, p) = c * vp - sn * vq;
    V(i, q) = sn * vp + c * vq;
  }
  return true;
}

template <typename S>
Svd<S> jacobi_tall(const Matrix<S>& A) {
  const Index m = A.rows(), n = A.cols();
  Matrix<S> U = A, V = Matrix<S>::Identity(n, n);
  const double tol = 1e-15;
  const Index np = n + (n & 1);  // players; index n is a bye when n is odd
  std::vector<Index> ring(static_cast<size_t>(np));
  const bool par = static_cast<double>(m) * n * n > 4e6;
  for (int sweep = 0; sweep < 80; ++sweep) {
    std::iota(ring.begin(), ring.end(), Index{0});
    int rotated = 0;
    for (Index round = 0; round + 1 < np; ++round) {
#pragma omp parallel for schedule(static) reduction(+ : rotated) if (par)
      for (Index k = 0; k < np / 2; ++k) {
        Index p = ring[static_cast<size_t>(k)], q = ring[static_cast<size_t>(np - 1 - k)];
        if (p > q) std::swap(p, q);
        if (q < n) rotated += rotate_pair(U, V, p, q, tol) ? 1 : 0;
      }
      std::rotate(ring.begin() + 1, ring.end() - 1, ring.end());  // circle method
    }
    if (!rotated) break;
  }
  std::vector<double> s(static_cast<size_t>(n));
  for (Index j = 0; j < n; ++j) {
    double t = 0.0;
    for (Index i = 0; i < m; ++i) t += abs2(U(i, j));
    s[j] = std::sqrt(t);
    if (s[j] > 0.0)
      for (Index i = 0; i < m; ++i) U(i, j) /= s[j];
  }
  std::vector<Index> ord(static_cast<size_t>(n));
  std::iota(ord.begin(), ord.end(), Index{0});
  std::stable_sort(ord.begin(), ord.end(), [&](Index x, Index y) { return s[x] > s[y]; });
  Svd<S> out;
  out.U = Matrix<S>(m, n);
  out.V = Matrix<S>(n, n);
  out.s.resize(static_cast<size_t>(n));
  for (Index j = 0; j < n; ++j) {
    const Index o = ord[j];
    out.s[j] = s[o];
    for (Index i = 0; i < m; ++i) out.U(i, j) = U(i, o);
    for (Index i = 0; i < n; ++i) out.V(i, j) = V(i, o);
  }
  return out;
}

template <typename S>
Svd<S> svd_impl(const Matrix<S>& A) {
  if (A.rows() >= A.cols()) return jacobi_tall(A);
  Svd<S> t = jacobi_tall(adjoint(A));  // A^H = U S V^H  =>  A = V S U^H
  return Svd<S>{std::move(t.V), std::move(t.s), std::move(t.U)};
}

// Householder QR without pivoting; Q = H_0 ... H_{r-1} [I; 0] (m x r).
template <typename S>
Matrix<S> thin_q_impl(const Matrix<S>& A0) {
  Matrix<S> A = A0;
  const Index m = A.rows(), n = A.cols(), r = std::min(m, n);
  std::vector<double> beta(static_cast<size_t>(r), 0.0);
  for (Index k = 0; k < r; ++k) {
    double xs = 0.0;
    for (Index i = k; i < m; ++i) xs += abs2(A(i, k));
    const double xn = std::sqrt(xs);
    if (xn == 0.0) continue;  // H_k = I
    const S a0 = A(k, k);
    const double aa = std::sqrt(abs2(a0));
    const S ph = aa == 0.0 ? S(1) : a0 / aa;
    const S v0 = a0 + ph * xn;
    double vs = 0.0;
    for (Index i = k + 1; i < m; ++i) {
      A(i, k) /= v0;
      vs += abs2(A(i, k));
    }
    beta[k] = 2.0 / (1.0 + vs);
    A(k, k) = -ph * xn;
    for (Index j = k + 1; j < n; ++j) {
      S w = A(k, j);
      for (Index i = k + 1; i < m; ++i) w += conj(A(i, k)) * A(i, j);
      w *= beta[k];
      A(k, j) -= w;
      for (Index i = k + 1; i < m; ++i) A(i, j) -= A(i, k) * w;
    }
  }
  Matrix<S> Q = Matrix<S>::Identity(m, r);
  for (Index k = r - 1; k >= 0; --k) {
    if (beta[k] == 0.0) continue;
    for (Index j = k; j < r; ++j) {
      S w = Q(k, j);
      for (Index i = k + 1; i < m; ++i) w += conj(A(i, k)) * Q(i, j);
      w *= beta[k];
      Q(k, j) -= w;
      for (Index i = k + 1; i < m; ++i) Q(i, j) -= A(i, k) * w;
    }
  }
  return Q;
}

template <typename S>
Matrix<S> pinv_impl(const Matrix<S>& A, double rel_cutoff, double* cond_out) {  // src/linalg.cpp:112-131
  const Svd<S> d = svd_impl(A);
  if (d.s.empty() || d.s[0] == 0.0) {
    if (cond_out) *cond_out = std::numeric_limits<double>::infinity();
    return Matrix<S>(A.cols(), A.rows());
  }
  if (cond_out) *cond_out = d.s[0] / std::max(d.s.back(), std::numeric_limits<double>::min());
  Matrix<S> P(A.cols(), A.rows());
  for (size_t l = 0; l < d.s.size(); ++l) {
    if (!(d.s[l] > rel_cutoff * d.s[0])) continue;
    const double inv = 1.0 / d.s[l];
    for (Index j = 0; j < A.rows(); ++j) {
      const S u = conj(d.U(j, static_cast<Index>(l))) * inv;
      for (Index i = 0; i < A.cols(); ++i) P(i, j) += d.V(i, static_cast<Index>(l)) * u;
    }
  }
  return P;
}

// Pivot order + completed steps of the reference's pqr_impl (src/linalg.cpp:23-107)
// on the complex embedding (identical arithmetic for real data).
template <typename S>
PivotedQR pqr_perm(const Matrix<S>& A, Index max_rank) {
  MatXc C(A.rows(), A.cols());
  for (Index i = 0; i < A.size(); ++i) C(i) = Cplx(A(i));
  return pivoted_qr(C, max_rank);
}

template <typename S>
RsvdResult<S> rsvd_impl(const SampledMatrix<S>& A, const IndexVec& R0, const IndexVec& C0, Index r,
                        std::mt19937_64& rng) {
  const Index m = A.rows, n = A.cols;
  const Index s = static_cast<Index>(R0.size());
  if (static_cast<Index>(C0.size()) != s) throw std::invalid_argument("rsvd: row and column samples differ in size");
  RsvdResult<S> out;
  std::unordered_map<Index, Matrix<S>> row_cache, col_cache;
  auto get_row = [&](Index i) -> const Matrix<S>& {
    auto it = row_cache.find(i);
    if (it == row_cache.end()) {
      ++out.rows_evaluated;
      Matrix<S> v = A.row(i);
      if (v.size() != n) throw std::invalid_argument("rsvd: row accessor returned a wrong length");
      it = row_cache.emplace(i, std::move(v)).first;
    }
    return it->second;
  };
  auto get_col = [&](Index j) -> const Matrix<S>& {
    auto it = col_cache.find(j);
    if (it == col_cache.end()) {
      ++out.cols_evaluated;
      Matrix<S> v = A.col(j);
      if (v.size() != m) throw std::invalid_argument("rsvd: column accessor returned a wrong length");
      it = col_cache.emplace(j, std::move(v)).first;
    }
    return it->second;
  };

  Matrix<S> rows_slab(s, n);
  for (Index i = 0; i < s; ++i) {
    const Matrix<S>& v = get_row(R0[i]);
    for (Index j = 0; j < n; ++j) rows_slab(i, j) = v(j);
  }
  const PivotedQR qr_c = pqr_perm(rows_slab, s);
  const Index sc = std::min<Index>(s, qr_c.rank);

  Matrix<S> cols_slab(m, s);
  for (Index j = 0; j < s; ++j) {
    const Matrix<S>& v = get_col(C0[j]);
    for (Index i = 0; i < m; ++i) cols_slab(i, j) = v(i);
  }
  const PivotedQR qr_r = pqr_perm(adjoint(cols_slab), s);
  const Index sr = std::min<Index>(s, qr_r.rank);

  if (sc == 0 || sr == 0) {
    out.U = Matrix<S>(m, 0);
    out.S = VecXd(0, 1);
    out.V = Matrix<S>(n, 0);
    return out;
  }
  const IndexVec pc(qr_c.perm.begin(), qr_c.perm.begin() + sc);
  const IndexVec pr(qr_r.perm.begin(), qr_r.perm.begin() + sr);

  Matrix<S> col_skel(m, sc);
  for (Index j = 0; j < sc; ++j) {
    const Matrix<S>& v = get_col(pc[j]);
    for (Index i = 0; i < m; ++i) col_skel(i, j) = v(i);
  }
  const Matrix<S> Q_col = thin_q_impl(col_skel);
  Matrix<S> row_skel_h(n, sr);  // row_skel^H
  for (Index i = 0; i < sr; ++i) {
    const Matrix<S>& v = get_row(pr[i]);
    for (Index j = 0; j < n; ++j) row_skel_h(j, i) = conj(v(j));
  }
  const Matrix<S> Q_row = thin_q_impl(row_skel_h);

  IndexVec I = pr, J = pc;
  for (Index i : rand_subset(m, sr, rng)) I.push_back(i);
  for (Index j : rand_subset(n, sc, rng)) J.push_back(j);

  Matrix<S> QcI(static_cast<Index>(I.size()), Q_col.cols());
  for (size_t i = 0; i < I.size(); ++i)
    for (Index c = 0; c < Q_col.cols(); ++c) QcI(static_cast<Index>(i), c) = Q_col(I[i], c);
  Matrix<S> QrJh(Q_row.cols(), static_cast<Index>(J.size()));  // QrJ^H
  for (size_t j = 0; j < J.size(); ++j)
    for (Index c = 0; c < Q_row.cols(); ++c) QrJh(c, static_cast<Index>(j)) = conj(Q_row(J[j], c));
  Matrix<S> AIJ(static_cast<Index>(I.size()), static_cast<Index>(J.size()));
  for (size_t i = 0; i < I.size(); ++i) {
    const Matrix<S>& v = get_row(I[i]);
    for (size_t j = 0; j < J.size(); ++j) AIJ(static_cast<Index>(i), static_cast<Index>(j)) = v(J[j]);
  }
  double cond_c = 0.0, cond_r = 0.0;
  const Matrix<S> M = matmul(matmul(pinv_impl(QcI, 1e-12, &cond_c), AIJ), pinv_impl(QrJh, 1e-12, &cond_r));
  out.ill_conditioned = !(cond_c < 1e8) || !(cond_r < 1e8);

  const Svd<S> d = svd_impl(M);
  const Index rr = std::min<Index>(r, static_cast<Index>(d.s.size()));
  Matrix<S> Ur(d.U.rows(), rr), Vr(d.V.rows(), rr);
  for (Index c = 0; c < rr; ++c) {
    for (Index i = 0; i < d.U.rows(); ++i) Ur(i, c) = d.U(i, c);
    for (Index i = 0; i < d.V.rows(); ++i) Vr(i, c) = d.V(i, c);
  }
  out.U = matmul(Q_col, Ur);
  out.V = matmul(Q_row, Vr);
  out.S = VecXd(rr, 1);
  for (Index c = 0; c < rr; ++c) out.S(c) = d.s[c];
  return out;
}

}  // namespace

MatXd thin_q(const MatXd& A) { return thin_q_impl(A); }
MatXc thin_q(const MatXc& A) { return thin_q_impl(A); }
MatXd pinv(const MatXd& A, double rel_cutoff, double* cond_out) { return pinv_impl(A, rel_cutoff, cond_out); }
MatXc pinv(const MatXc& A, double rel_cutoff, double* cond_out) { return pinv_impl(A, rel_cutoff, cond_out); }
Svd<double> svd(const MatXd& A) { return svd_impl(A); }
Svd<Cplx> svd(const MatXc& A) { return svd_impl(A); }
RsvdResult<double> rsvd(const SampledMatrix<double>& A, const IndexVec& R0, const IndexVec& C0, Index r,
                        std::mt19937_64& rng) {
  return rsvd_impl(A, R0, C0, r, rng);
}
RsvdResult<Cplx> rsvd(const SampledMatrix<Cplx>& A, const IndexVec& R0, const IndexVec& C0, Index r,
                      std::mt19937_64& rng) {
  return rsvd_impl(A, R0, C0, r, rng);
}

}  // namespace midbf::la

namespace midbf::phase {

PhaseAccessorMD explicit_phase_accessor(const ker::KernelDesc& K) {
  auto smp = std::make_shared<dev::EntrySampler>(K);
  PhaseAccessorMD acc;
  acc.nrows = K.nrows;
  acc.ncols = K.ncols;
  acc.row = [smp, K](Index i) {
    VecXd v(K.ncols, 1);
    smp->phase_block(1, &i, K.ncols, nullptr, v.data());
    return v;
  };
  acc.col = [smp, K](Index j) {
    VecXd v(K.nrows, 1);
    smp->phase_block(K.nrows, nullptr, 1, &j, v.data());
    return v;
  };
  return acc;
}

PhaseFactorization low_rank_phase_factorization(const PhaseAccessorMD& acc, Index r, Index q_oversample,
                                                std::mt19937_64& rng) {
  const Index n1 = acc.nrows, n2 = acc.ncols;
  const Index s = r * q_oversample;
  if (r < 1 || q_oversample < 1) throw std::invalid_argument("rank and oversampling must be positive");
  if (s > n1 || s > n2) throw std::invalid_argument("sample budget r*q exceeds the matrix size");
  const IndexVec R = la::rand_subset(n1, s, rng);  // src/phase_md.cpp:198-199
  const IndexVec C = la::rand_subset(n2, s, rng);
  la::SampledMatrix<double> A{n1, n2, acc.row, acc.col};
  la::RsvdResult<double> svd = la::rsvd(A, R, C, r, rng);
  PhaseFactorization out;  // :211-217
  out.phase.U = std::move(svd.U);
  out.phase.V = MatXd(svd.V.rows(), svd.V.cols());
  for (Index c = 0; c < svd.V.cols(); ++c)
    for (Index i = 0; i < svd.V.rows(); ++i) out.phase.V(i, c) = svd.V(i, c) * svd.S(c);
  out.rows_evaluated = svd.rows_evaluated;
  out.cols_evaluated = svd.cols_evaluated;
  return out;
}

}  // namespace midbf::phase

namespace midbf::metrics {

double eps_K(const phase::LowRankPhase& ph, const ker::KernelDesc& K, Index nsamp, std::uint64_t seed) {
  const Index nr = ph.U.rows(), nc = ph.V.rows(), r = ph.U.cols();
  if (nsamp < 1) throw std::invalid_argument("eps_K: need at least one sample");
  if (ph.V.cols() != r || nr != K.nrows || nc != K.ncols)
    throw std::invalid_argument("eps_K: phase factors do not match the kernel");
  std::mt19937_64 rng(seed);  // src/metrics.cpp:61-71
  auto draw = [&rng, nsamp](Index n) {
    IndexVec S;
    if (nsamp >= n) {
      S.resize(static_cast<size_t>(n));
      std::iota(S.begin(), S.end(), Index{0});
    } else {
      S = la::rand_subset(n, nsamp, rng);
    }
    return S;
  };
  const IndexVec S1 = draw(nr), S2 = draw(nc);
  const Index a = static_cast<Index>(S1.size()), b = static_cast<Index>(S2.size());
  // A = K(S1, S2), B = exp(2 pi i U(S1) V(S2)^T): both on the GPU (K3)
  const std::int64_t task[5] = {0, a, 0, b, 0};
  MatXc A(a, b), B(a, b);
  dev::EntrySampler(K).sample(1, task, S1.data(), a, S2.data(), b, reinterpret_cast<double*>(A.data()), a * b);
  std::vector<double> Ur(static_cast<size_t>(nr * r)), Vr(static_cast<size_t>(nc * r));  // row-major factors
  for (Index i = 0; i < nr; ++i)
    for (Index c = 0; c < r; ++c) Ur[static_cast<size_t>(i * r + c)] = ph.U(i, c);
  for (Index j = 0; j < nc; ++j)
    for (Index c = 0; c < r; ++c) Vr[static_cast<size_t>(j * r + c)] = ph.V(j, c);
  ker::KernelDesc L{};
  L.kind = MIDBF_KERNEL_LOWRANK;
  L.rank = static_cast<std::int32_t>(r);
  L.nrows = nr;
  L.ncols = nc;
  L.A = Ur.data();
  L.B = Vr.data();
  if (r > 0) {
    dev::EntrySampler(L).sample(1, task, S1.data(), a, S2.data(), b, reinterpret_cast<double*>(B.data()), a * b);
  } else {
    for (Index i = 0; i < B.size(); ++i) B(i) = Cplx(1.0, 0.0);  // exp(0)
  }
  MatXc D(a, b);
  for (Index i = 0; i < D.size(); ++i) D(i) = A(i) - B(i);
  const double num = la::svd(D).s[0], den = la::svd(A).s[0];
  return den == 0.0 ? num : num / den;
}

}  // namespace midbf::metrics

// ------------------------------------------------------------------ C ABI
#include "../status.hpp"
#include "midbf_b200.h"

namespace {

using midbf::Cplx;
using midbf::Index;
using midbf::Matrix;

template <typename S>
Matrix<S> in_mat(const double* A, int64_t m, int64_t n) {
  Matrix<S> M(m, n);
  std::memcpy(static_cast<void*>(M.data()), A, static_cast<size_t>(m * n) * sizeof(S));
  return M;
}
template <typename S>
void out_mat(const Matrix<S>& M, double* out, int64_t rows, int64_t cols) {  // zero-padded to rows x cols
  S* o = reinterpret_cast<S*>(out);
  std::fill(o, o + rows * cols, S(0));
  for (Index j = 0; j < std::min<Index>(cols, M.cols()); ++j)
    for (Index i = 0; i < std::min<Index>(rows, M.rows()); ++i) o[i + j * rows] = M(i, j);
}

template <typename S>
void rsvd_dense(const double* A, int64_t m, int64_t n, const int64_t* R0, const int64_t* C0, int64_t s, int64_t r,
                uint64_t seed, double* U, double* Sv, double* V, int64_t* info) {
  const Matrix<S> M = in_mat<S>(A, m, n);
  midbf::la::SampledMatrix<S> sm;
  sm.rows = m;
  sm.cols = n;
  sm.row = [&M, n](Index i) {
    Matrix<S> v(n, 1);
    for (Index j = 0; j < n; ++j) v(j) = M(i, j);
    return v;
  };
  sm.col = [&M, m](Index j) {
    Matrix<S> v(m, 1);
    for (Index i = 0; i < m; ++i) v(i) = M(i, j);
    return v;
  };
  for (int64_t q = 0; q < s; ++q)
    if (R0[q] < 0 || R0[q] >= m || C0[q] < 0 || C0[q] >= n) throw std::invalid_argument("sample index out of range");
  std::mt19937_64 rng(seed);
  const auto res = midbf::la::rsvd(sm, midbf::IndexVec(R0, R0 + s), midbf::IndexVec(C0, C0 + s), r, rng);
  out_mat(res.U, U, m, r);
  out_mat(res.V, V, n, r);
  for (int64_t c = 0; c < r; ++c) Sv[c] = c < res.S.size() ? res.S(c) : 0.0;
  info[0] = res.S.size();
  info[1] = res.rows_evaluated;
  info[2] = res.cols_evaluated;
  info[3] = res.ill_conditioned ? 1 : 0;
}

}  // namespace

extern "C" int midbf_thin_q(const double* A, int64_t m, int64_t n, int is_complex, double* Q) {
  return midbf::detail::guard([&] {
    if (m < 0 || n < 0 || (m * n > 0 && (!A || !Q))) throw std::invalid_argument("bad arguments");
    const int64_t r = std::min(m, n);
    if (is_complex)
      out_mat(midbf::la::thin_q(in_mat<Cplx>(A, m, n)), Q, m, r);
    else
      out_mat(midbf::la::thin_q(in_mat<double>(A, m, n)), Q, m, r);
  });
}

extern "C" int midbf_pinv(const double* A, int64_t m, int64_t n, int is_complex, double rel_cutoff, double* P,
                          double* cond) {
  return midbf::detail::guard([&] {
    if (m < 0 || n < 0 || (m * n > 0 && (!A || !P))) throw std::invalid_argument("bad arguments");
    double c = 0.0;
    if (is_complex)
      out_mat(midbf::la::pinv(in_mat<Cplx>(A, m, n), rel_cutoff, &c), P, n, m);
    else
      out_mat(midbf::la::pinv(in_mat<double>(A, m, n), rel_cutoff, &c), P, n, m);
    if (cond) *cond = c;
  });
}

extern "C" int midbf_rsvd_dense(const double* A, int64_t m, int64_t n, int is_complex, const int64_t* R0,
                                const int64_t* C0, int64_t s, int64_t r, uint64_t seed, double* U, double* S,
                                double* V, int64_t* info) {
  return midbf::detail::guard([&] {
    if (m <= 0 || n <= 0 || s <= 0 || r <= 0 || !A || !R0 || !C0 || !U || !S || !V || !info)
      throw std::invalid_argument("bad arguments");
    if (is_complex)
      rsvd_dense<Cplx>(A, m, n, R0, C0, s, r, seed, U, S, V, info);
    else
      rsvd_dense<double>(A, m, n, R0, C0, s, r, seed, U, S, V, info);
  });
}

extern "C" int midbf_lowrank_phase(const midbf_kernel_desc* kernel, int64_t r, int64_t q, uint64_t seed, double* U,
                                   double* V, int64_t* info) {
  return midbf::detail::guard([&] {
    if (!kernel || !U || !V || !info) throw std::invalid_argument("null argument");
    std::mt19937_64 rng(seed);
    const auto pf =
        midbf::phase::low_rank_phase_factorization(midbf::phase::explicit_phase_accessor(*kernel), r, q, rng);
    out_mat(pf.phase.U, U, kernel->nrows, r);
    out_mat(pf.phase.V, V, kernel->ncols, r);
    info[0] = pf.phase.U.cols();
    info[1] = pf.rows_evaluated;
    info[2] = pf.cols_evaluated;
  });
}

extern "C" int midbf_eps_K(const midbf_kernel_desc* kernel, const double* U, const double* V, int64_t r,
                           int64_t nsamp, uint64_t seed, double* out) {
  return midbf::detail::guard([&] {
    if (!kernel || !out || r < 0 || (r > 0 && (!U || !V))) throw std::invalid_argument("null argument");
    midbf::phase::LowRankPhase ph;
    ph.U = in_mat<double>(U, kernel->nrows, r);
    ph.V = in_mat<double>(V, kernel->ncols, r);
    *out = midbf::metrics::eps_K(ph, *kernel, nsamp, seed);
  });
}
