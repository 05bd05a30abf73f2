// Low-rank phase production: the sampling-based SVD
// la::rsvd with its helpers thin_q / pinv (reference
// proj/include/midbf/linalg.hpp:27-61, src/linalg.cpp:109-219), the low-rank
// phase factorization (include/midbf/phase_md.hpp:104-126,
// src/phase_md.cpp:184-224) for phases available in closed form, and the
// phase accuracy metric eps_K (include/midbf/metrics.hpp, src/metrics.cpp:55-86).
//
// Explicit phases only: the reference's RecoveredMatrixMD unwraps mod-1
// observations along Delaunay/MST recovery paths (src/phase_md.cpp:63-152,
// src/geometry.cpp, src/delaunay.cpp) — out of scope.  For a
// phase given in closed form (FIO 2D/3D, x.xi, A.B^T) recovery is the
// identity, so low_rank_phase_factorization feeds the sampled rows/columns
// straight to rsvd; rows and columns of Phi are evaluated on the GPU.
#pragma once

#include <cstdint>
#include <functional>
#include <random>

#include "midbf/kernels.hpp"
#include "midbf/types.hpp"

namespace midbf::la {

// Orthonormal basis of range(A) (m x min(m,n)), Householder QR (:27-28).
MatXd thin_q(const MatXd& A);
MatXc thin_q(const MatXc& A);

// Moore-Penrose pseudoinverse through the SVD; singular values at or below
// rel_cutoff * sigma_max are treated as zero (:30-33).  cond_out (optional):
// sigma_max / sigma_min of the thin SVD.
MatXd pinv(const MatXd& A, double rel_cutoff = 1e-12, double* cond_out = nullptr);
MatXc pinv(const MatXc& A, double rel_cutoff = 1e-12, double* cond_out = nullptr);

// Singular values (descending) with thin U (m x p) and V (n x p), p = min(m,n)
// (one-sided Jacobi; the reference uses Eigen::JacobiSVD / BDCSVD).
template <typename Scalar>
struct Svd {
  Matrix<Scalar> U;
  std::vector<double> s;
  Matrix<Scalar> V;
};
Svd<double> svd(const MatXd& A);
Svd<Cplx> svd(const MatXc& A);

template <typename Scalar>
struct SampledMatrix {  // :35-43
  Index rows = 0;
  Index cols = 0;
  std::function<Matrix<Scalar>(Index)> row;  // length cols
  std::function<Matrix<Scalar>(Index)> col;  // length rows
};

template <typename Scalar>
struct RsvdResult {  // :45-53
  Matrix<Scalar> U;  // m x r
  VecXd S;           // r singular values
  Matrix<Scalar> V;  // n x r, A ~ U S V^H
  bool ill_conditioned = false;
  Index rows_evaluated = 0;
  Index cols_evaluated = 0;
};

// Randomized SVD from sampled rows R0 / columns C0 (equal sizes) (:55-61,
// src/linalg.cpp:134-219).
RsvdResult<double> rsvd(const SampledMatrix<double>& A, const IndexVec& R0, const IndexVec& C0, Index r,
                        std::mt19937_64& rng);
RsvdResult<Cplx> rsvd(const SampledMatrix<Cplx>& A, const IndexVec& R0, const IndexVec& C0, Index r,
                      std::mt19937_64& rng);

}  // namespace midbf::la

namespace midbf::phase {

struct PhaseAccessorMD {  // include/midbf/phase_md.hpp:24-29 (explicit phase values)
  Index nrows = 0;
  Index ncols = 0;
  std::function<VecXd(Index)> row;  // length ncols
  std::function<VecXd(Index)> col;  // length nrows
};

struct LowRankPhase {  // :104-107
  MatXd U;  // nrows x r
  MatXd V;  // ncols x r
};

struct PhaseFactorization {  // :109-116
  LowRankPhase phase;
  Index n_disc_rows = 0;
  Index n_disc_cols = 0;
  Index rows_evaluated = 0;
  Index cols_evaluated = 0;
  double tau = 0.25;
};

// Rows/columns of the closed-form phase of K, evaluated on the GPU.
PhaseAccessorMD explicit_phase_accessor(const ker::KernelDesc& K);

// src/phase_md.cpp:184-224 with recovery = identity: R = rand_subset(n1, r q),
// C = rand_subset(n2, r q) from rng, rsvd(Phi, R, C, r, rng), U <- U,
// V <- V * diag(S).
PhaseFactorization low_rank_phase_factorization(const PhaseAccessorMD& acc, Index r, Index q_oversample,
                                                std::mt19937_64& rng);

}  // namespace midbf::phase

namespace midbf::metrics {

// src/metrics.cpp:55-86: spectral-norm relative error between K(S1, S2) and
// exp(2 pi i U(S1) V(S2)^T) on rand_subset rows/columns (all when
// nsamp >= n); both blocks sampled on the GPU.
double eps_K(const phase::LowRankPhase& ph, const ker::KernelDesc& K, Index nsamp, std::uint64_t seed);

}  // namespace midbf::metrics
