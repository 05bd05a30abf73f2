// TEST INFRASTRUCTURE ONLY — declarations of the CPU oracle (restatement of
// the reference MIDBF path, see orc_core.cpp).  Not part of the product.
#pragma once

#include <array>
#include <functional>
#include <random>
#include <string>
#include <utility>

#include "orc_mat.hpp"

namespace orc {

std::uint64_t mix64(std::uint64_t x);
std::uint64_t chain(std::uint64_t a, std::uint64_t b);

// include/midbf/tree.hpp:12-34
struct Node {
  std::uint64_t code = 0;
  Index parent = -1;
  Index begin = 0, end = 0;
  std::array<Index, 8> child{{-1, -1, -1, -1, -1, -1, -1, -1}};
  Index nchild = 0;
};
struct Tree {
  int dim = 2;
  Index n0 = 0;
  int depth = 0;
  std::vector<std::vector<Node>> levels;
  IndexVec perm;
};
Tree build_tree(const MatXd& X, Index n0, int min_depth);

// include/midbf/linalg.hpp:13-20
template <class S>
struct QR {
  Mat<S> Q, R;
  IndexVec perm;
  Index rank = 0;
};
template <class S>
QR<S> pivoted_qr(Mat<S> A, Index max_rank);

struct ColumnID {
  IndexVec skeleton;
  MatXc V;
  Index rank = 0;
};
struct RowID {
  IndexVec skeleton;
  MatXc W;
  Index rank = 0;
};
Index id_rank(const std::vector<double>& dg, Index k_max, double eps);
ColumnID cid_from_rows(const MatXc& blk, Index k_max, double eps);
RowID rid_from_cols(const MatXc& blk, Index k_max, double eps);
IndexVec mock_chebyshev_rows(const std::vector<double>& pts, Index s);
IndexVec mock_chebyshev_points(const MatXd& P, Index s, std::mt19937_64& rng);
IndexVec rand_subset(Index n, Index k, std::mt19937_64& rng);

// include/midbf/butterfly.hpp:24-70
using EntryFn = std::function<Cplx(Index, Index)>;
struct Block {
  Index row_off = 0, col_off = 0;
  MatXc M;
};
struct Factor {
  Index rows = 0, cols = 0;
  std::vector<Block> blocks;
  std::vector<std::pair<Index, Index>> groups;
};
struct Config {
  Index k_max = 30;
  double eps = 1e-9;
  Index t = 5;
  std::uint64_t seed = 0;
  bool parallel = false;
};
struct Factorization {
  Index nrows = 0, ncols = 0;
  int L = 0, h = 0;
  Index n0 = 0;
  Config cfg;
  IndexVec row_perm, col_perm;
  std::vector<Factor> factors;
  Index total_nnz() const;
  Index max_factor_nnz() const;
  double nnz_bound(double c) const;
};

Factorization idbf_factorize(const EntryFn& K, const Tree& tx, const Tree& to, const MatXd& X,
                             const MatXd& Om, const Config& cfg);
void apply(const Factorization& F, const Cplx* in, Index nrhs, bool tr, Cplx* out, bool par);
void save(const std::string& path, const Factorization& F);
Factorization load(const std::string& path);

// Kernel descriptions (shared numbering with the product's midbf_kernel_desc).
enum Kind { KIND_FIO2D = 0, KIND_FIO3D = 1, KIND_LOWRANK = 2, KIND_NUFFT = 3, KIND_CONST = 4, KIND_RANK1 = 5 };
struct KernelDesc {
  int kind = KIND_FIO2D;
  int dim = 2;
  int rank = 0;
  Index nrows = 0, ncols = 0;
  const double* X = nullptr;
  const double* Omega = nullptr;
  const double* A = nullptr;
  const double* B = nullptr;
  const double* u = nullptr;
  const double* v = nullptr;
  double cre = 0, cim = 0;
};
double fio2d_phase(const double* x, const double* xi);
double fio3d_phase(const double* x, const double* xi);
EntryFn make_entry(const KernelDesc& kd);
void direct_sum(const EntryFn& K, Index ncols, const Cplx* f, const Index* rows, Index nrows, Cplx* out, bool par);
double eps_b_of(const Cplx* gb, Index N, const EntryFn& K, const Cplx* f, Index n, Index nrows, std::uint64_t seed);
void random_coefficients(Index n, std::uint64_t seed, Cplx* out);
void grid2d(Index n, double* X);

}  // namespace orc
