// TEST INFRASTRUCTURE ONLY — a C ABI over the REFERENCE's own MIDBF code,
// compiled unmodified from /root/reference/proj/src against the Eigen
// stand-in in oracle/shim/ (oracle/ref.mk builds oracle/_ref/libmidbf_ref.so).
// tests/ use it (through oracle/ref.py) to pin the oracle restatement
// (orc_core.cpp) and the product's host factorize against the reference,
// and tests/golden/make_golden.py generates the committed fixtures with it.
// Nothing here is reference source: every call goes to the reference API
// (proj/include/midbf/*.hpp).  The one kernel the reference lacks, BASELINE
// cfg3's 3D phase, is written here in the operation order of the 2D
// fio2d_phase (src/kernels.cpp:18-24) — the same restatement the oracle and
// the product use (oracle/orc_core.cpp fio3d_phase).
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "midbf/butterfly.hpp"
#include "midbf/butterfly_io.hpp"
#include "midbf/geometry.hpp"
#include "midbf/kernels.hpp"
#include "midbf/linalg.hpp"
#include "midbf/metrics.hpp"
#include "midbf/phase_md.hpp"
#include "midbf/tree.hpp"

using namespace midbf;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return -2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -3;
  }
}

// kinds shared with oracle/oracle.py
enum { KIND_FIO2D, KIND_FIO3D, KIND_LOWRANK, KIND_NUFFT, KIND_CONST, KIND_RANK1 };
constexpr double kTwoPi = 6.283185307179586476925286766559;

MatXd points(const double* P, std::int64_t n, int dim) {  // row-major in, MatXd out
  MatXd M(n, dim);
  for (std::int64_t i = 0; i < n; ++i)
    for (int d = 0; d < dim; ++d) M(i, d) = P[i * dim + d];
  return M;
}

double fio3d_phase(const double* x, const double* xi) {  // BASELINE configs[3]
  const double s0 = std::sin(kTwoPi * x[0]), s1 = std::sin(kTwoPi * x[1]), s2 = std::sin(kTwoPi * x[2]);
  const double c0 = std::cos(kTwoPi * x[0]), c1 = std::cos(kTwoPi * x[1]), c2 = std::cos(kTwoPi * x[2]);
  const double a1 = (2.0 + s0 * s1 * s2) / 16.0;
  const double a2 = (2.0 + c0 * c1 * c2) / 16.0;
  const double a3 = (2.0 + s0 * c1 * s2) / 16.0;
  return x[0] * xi[0] + x[1] * xi[1] + x[2] * xi[2] +
         std::sqrt(a1 * a1 * xi[0] * xi[0] + a2 * a2 * xi[1] * xi[1] + a3 * a3 * xi[2] * xi[2]);
}

struct Kern {
  bf::EntryFn K;
  std::shared_ptr<MatXd> X, O;
};

Kern make_kernel(int kind, const double* X, std::int64_t nx, const double* Om, std::int64_t no, int dim,
                 const double* A, const double* B, int rank, const double* cst, const double* u, const double* v) {
  Kern k;
  if (X) {
    k.X = std::make_shared<MatXd>(points(X, nx, dim));
    k.O = std::make_shared<MatXd>(points(Om, no, dim));
  }
  switch (kind) {
    case KIND_FIO2D:  // the reference's scenario-1 accessor (src/kernels.cpp:228-245)
      k.K = ker::make_accessor(ker::KernelKind::Fio2D, *k.X, *k.O, 1).entry;
      break;
    case KIND_NUFFT:
      k.K = ker::make_accessor(ker::KernelKind::Nufft, *k.X, *k.O, 1).entry;
      break;
    case KIND_LOWRANK: {  // metrics::phase_entry_fn (src/metrics.cpp:18-24)
      phase::LowRankPhase ph;
      ph.U = points(A, nx, rank);
      ph.V = points(B, no, rank);
      k.K = metrics::phase_entry_fn(ph);
      break;
    }
    case KIND_FIO3D: {
      std::vector<double> xs(X, X + 3 * nx), os(Om, Om + 3 * no);
      auto px = std::make_shared<std::vector<double>>(std::move(xs));
      auto po = std::make_shared<std::vector<double>>(std::move(os));
      k.K = [px, po](Index i, Index j) {
        return std::polar(1.0, kTwoPi * fio3d_phase(px->data() + 3 * i, po->data() + 3 * j));
      };
      break;
    }
    case KIND_CONST: {
      const Cplx c(cst[0], cst[1]);
      k.K = [c](Index, Index) { return c; };
      break;
    }
    case KIND_RANK1: {
      auto pu = std::make_shared<std::vector<Cplx>>(reinterpret_cast<const Cplx*>(u),
                                                    reinterpret_cast<const Cplx*>(u) + nx);
      auto pv = std::make_shared<std::vector<Cplx>>(reinterpret_cast<const Cplx*>(v),
                                                    reinterpret_cast<const Cplx*>(v) + no);
      k.K = [pu, pv](Index i, Index j) { return (*pu)[i] * (*pv)[j]; };
      break;
    }
    default:
      throw std::invalid_argument("unknown kernel kind");
  }
  return k;
}

// Trees at a common depth, as the reference's tests build them
// (tests/test_butterfly.cpp:50-58 make_trees).
std::pair<tree::ClusterTree, tree::ClusterTree> make_trees(const MatXd& X, const MatXd& O, Index n0) {
  tree::ClusterTree tx = tree::build_tree(X, n0);
  tree::ClusterTree to = tree::build_tree(O, n0);
  const int L = std::max(tx.depth, to.depth);
  if (tx.depth != L) tx = tree::build_tree(X, n0, L);
  if (to.depth != L) to = tree::build_tree(O, n0, L);
  return {std::move(tx), std::move(to)};
}

}  // namespace

// src/delaunay.cpp needs gmpxx (absent here) and belongs to the phase-recovery
// geometry, which is out of scope; its one entry point is
// defined to fail loudly so that the library resolves.
namespace midbf::geo {
Triangulation delaunay_cells(const MatXd&) {
  throw std::runtime_error("delaunay_cells: src/delaunay.cpp (gmpxx) is not built in oracle/_ref");
}
}  // namespace midbf::geo

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// bf::idbf_factorize (src/butterfly.cpp:708-769) on the given points, saved
// with bf::save_factorization (src/butterfly_io.cpp:63-101).  Points are
// row-major (n, dim); for KIND_LOWRANK A / B are row-major (n, rank) and X /
// Om still give the tree geometry.
int ref_factorize(int kind, const double* X, std::int64_t nx, const double* Om, std::int64_t no, int dim,
                  const double* A, const double* B, int rank, const double* cst, const double* u, const double* v,
                  std::int64_t n0, std::int64_t k, double eps, std::int64_t t, std::uint64_t seed, int parallel,
                  const char* path) {
  return guard([&] {
    Kern kn = make_kernel(kind, X, nx, Om, no, dim, A, B, rank, cst, u, v);
    const MatXd XX = points(X, nx, dim), OO = points(Om, no, dim);
    auto tr = make_trees(XX, OO, n0);
    bf::Config cfg;
    cfg.rank = {k, eps};
    cfg.t = t;
    cfg.seed = seed;
    cfg.exec = parallel ? Exec::Parallel : Exec::Serial;
    const bf::Factorization F = bf::idbf_factorize(kn.K, tr.first, tr.second, XX, OO, cfg);
    bf::save_factorization(path, F);
  });
}

// bf::apply / bf::apply_transpose (src/butterfly.cpp:771-783) of a MIDBF001
// container on column-major (n, nrhs) complex input.
int ref_apply(const char* path, const double* f, std::int64_t n, std::int64_t nrhs, int transpose, double* out) {
  return guard([&] {
    const bf::Factorization F = bf::load_factorization(path);
    MatXc fs(n, nrhs);
    std::memcpy(fs.data(), f, sizeof(Cplx) * n * nrhs);
    const MatXc g = transpose ? bf::apply_transpose(F, fs) : bf::apply(F, fs);
    std::memcpy(out, g.data(), sizeof(Cplx) * g.rows() * g.cols());
  });
}

// A loaded factorization for repeated applies (bench.py's reference arm
// times bf::apply alone, not the container read).
int ref_load(const char* path, void** out) {
  return guard([&] { *out = new bf::Factorization(bf::load_factorization(path)); });
}
void ref_free(void* h) { delete static_cast<bf::Factorization*>(h); }
int ref_apply_h(void* h, const double* f, std::int64_t n, std::int64_t nrhs, int transpose, double* out) {
  return guard([&] {
    const bf::Factorization& F = *static_cast<bf::Factorization*>(h);
    MatXc fs(n, nrhs);
    std::memcpy(fs.data(), f, sizeof(Cplx) * n * nrhs);
    const MatXc g = transpose ? bf::apply_transpose(F, fs) : bf::apply(F, fs);
    std::memcpy(out, g.data(), sizeof(Cplx) * g.rows() * g.cols());
  });
}

// nrows ncols L h n0 nfactors total_nnz max_factor_nnz
int ref_info(const char* path, std::int64_t* o) {
  return guard([&] {
    const bf::Factorization F = bf::load_factorization(path);
    o[0] = F.nrows;
    o[1] = F.ncols;
    o[2] = F.L;
    o[3] = F.h;
    o[4] = F.n0;
    o[5] = F.factor_count();
    o[6] = F.total_nnz();
    o[7] = F.max_factor_nnz();
  });
}

// Kernel entries K(rows[q], cols[q]) through the reference's evaluators.
int ref_entries(int kind, const double* X, std::int64_t nx, const double* Om, std::int64_t no, int dim,
                const double* A, const double* B, int rank, const std::int64_t* rows, const std::int64_t* cols,
                std::int64_t n, double* out) {
  return guard([&] {
    Kern kn = make_kernel(kind, X, nx, Om, no, dim, A, B, rank, nullptr, nullptr, nullptr);
    for (std::int64_t q = 0; q < n; ++q) {
      const Cplx e = kn.K(rows[q], cols[q]);
      out[2 * q] = e.real();
      out[2 * q + 1] = e.imag();
    }
  });
}

// Direct sum g(rows[q]) = sum_j K(rows[q], j) f(j) through the reference's
// entry evaluator, accumulated in the loop order of src/metrics.cpp:40-43
// (= tests/test_butterfly.cpp:29-37 dense_matvec).
int ref_direct_sum(int kind, const double* X, std::int64_t nx, const double* Om, std::int64_t no, int dim,
                   const double* A, const double* B, int rank, const double* f, const std::int64_t* rows,
                   std::int64_t nr, double* out) {
  return guard([&] {
    Kern kn = make_kernel(kind, X, nx, Om, no, dim, A, B, rank, nullptr, nullptr, nullptr);
    const Cplx* fv = reinterpret_cast<const Cplx*>(f);
#pragma omp parallel for schedule(dynamic)
    for (std::int64_t q = 0; q < nr; ++q) {
      Cplx gd(0.0, 0.0);
      for (std::int64_t j = 0; j < no; ++j) gd += kn.K(rows[q], j) * fv[j];
      out[2 * q] = gd.real();
      out[2 * q + 1] = gd.imag();
    }
  });
}

// metrics::eps_b (src/metrics.cpp:26-53): apply + direct sum on sampled rows.
int ref_eps_b(const char* path, int kind, const double* X, std::int64_t nx, const double* Om, std::int64_t no, int dim,
              const double* A, const double* B, int rank, const double* f, std::int64_t nrows, std::uint64_t seed,
              double* out) {
  return guard([&] {
    Kern kn = make_kernel(kind, X, nx, Om, no, dim, A, B, rank, nullptr, nullptr, nullptr);
    const bf::Factorization F = bf::load_factorization(path);
    VecXc fv(F.ncols);
    std::memcpy(fv.data(), f, sizeof(Cplx) * F.ncols);
    *out = metrics::eps_b(F, kn.K, fv, nrows, seed);
  });
}

// tree::build_tree (src/tree.cpp:30-114): perm and depth.
int ref_tree(const double* X, std::int64_t n, int dim, std::int64_t n0, int min_depth, std::int64_t* perm,
             std::int64_t* depth) {
  return guard([&] {
    const tree::ClusterTree T = tree::build_tree(points(X, n, dim), n0, min_depth);
    for (std::int64_t i = 0; i < n; ++i) perm[i] = T.perm[static_cast<size_t>(i)];
    *depth = T.depth;
  });
}

// la::pivoted_qr (src/linalg.cpp:23-107) of a column-major complex (m, n)
// block: perm (n), rank, and R (rank x n, column-major) if R is non-null.
int ref_pqr(const double* a, std::int64_t m, std::int64_t n, std::int64_t max_rank, std::int64_t* perm,
            std::int64_t* rank, double* R) {
  return guard([&] {
    MatXc A(m, n);
    std::memcpy(A.data(), a, sizeof(Cplx) * m * n);
    const la::PivotedQR<Cplx> qr = la::pivoted_qr(A, max_rank);
    for (std::int64_t j = 0; j < n; ++j) perm[j] = qr.perm[static_cast<size_t>(j)];
    *rank = qr.rank;
    if (R) std::memcpy(R, qr.R.data(), sizeof(Cplx) * qr.R.rows() * qr.R.cols());
  });
}

// la::cid_from_rows (src/linalg.cpp:266-286): skeleton (rank) and V (rank x n).
int ref_cid(const double* a, std::int64_t m, std::int64_t n, std::int64_t k_max, double eps, std::int64_t* skel,
            double* V, std::int64_t* rank) {
  return guard([&] {
    MatXc A(m, n);
    std::memcpy(A.data(), a, sizeof(Cplx) * m * n);
    const la::ColumnID id = la::cid_from_rows(A, la::RankSpec{k_max, eps});
    *rank = id.rank;
    for (std::int64_t i = 0; i < id.rank; ++i) skel[i] = id.skeleton[static_cast<size_t>(i)];
    std::memcpy(V, id.V.data(), sizeof(Cplx) * id.V.rows() * id.V.cols());
  });
}

// la::mock_chebyshev_points (src/linalg.cpp:329-388) with mt19937_64(seed).
std::int64_t ref_mock_cheb_points(const double* P, std::int64_t n, int dim, std::int64_t s, std::uint64_t seed,
                                  std::int64_t* out) {
  std::mt19937_64 rng(seed);
  const IndexVec v = la::mock_chebyshev_points(points(P, n, dim), s, rng);
  for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
  return static_cast<std::int64_t>(v.size());
}

// la::rand_subset (src/linalg.cpp:390-400) with mt19937_64(seed).
std::int64_t ref_rand_subset(std::int64_t n, std::int64_t k, std::uint64_t seed, std::int64_t* out) {
  std::mt19937_64 rng(seed);
  const IndexVec v = la::rand_subset(n, k, rng);
  for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
  return static_cast<std::int64_t>(v.size());
}

// ker::grid2d (src/kernels.cpp:37-45), row-major (n*n, 2) out.
void ref_grid2d(std::int64_t n, double* out) {
  const MatXd X = ker::grid2d(n);
  for (Index i = 0; i < X.rows(); ++i)
    for (Index d = 0; d < 2; ++d) out[2 * i + d] = X(i, d);
}

}  // extern "C"
