// TEST INFRASTRUCTURE ONLY — flat C entry points of the CPU oracle for the
// Python tests (ctypes).  Exceptions become negative status codes with the
// message kept for orc_last_error(): -1 std::invalid_argument, -2
// std::logic_error, -3 std::runtime_error / other.
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "orc_core.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& fn) {
  try {
    fn();
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

MatXd points(const double* P, Index n, int dim) {  // row-major n x dim -> Mat
  MatXd M(n, dim);
  for (Index i = 0; i < n; ++i)
    for (int a = 0; a < dim; ++a) M(i, a) = P[i * dim + a];
  return M;
}

template <class S>
Mat<S> from_colmajor(const double* A, Index m, Index n) {
  Mat<S> M(m, n);
  std::memcpy(static_cast<void*>(M.d.data()), A, sizeof(S) * static_cast<size_t>(m * n));
  return M;
}

// tests/test_butterfly.cpp:52-60: both trees at the deeper common depth.
std::pair<Tree, Tree> make_trees(const MatXd& X, const MatXd& O, Index n0) {
  Tree tx = build_tree(X, n0, 0), to = build_tree(O, n0, 0);
  const int L = std::max(tx.depth, to.depth);
  if (tx.depth != L) tx = build_tree(X, n0, L);
  if (to.depth != L) to = build_tree(O, n0, L);
  return {std::move(tx), std::move(to)};
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
std::uint64_t orc_chain(std::uint64_t a, std::uint64_t b) { return chain(a, b); }

int orc_tree_build(const double* X, std::int64_t n, int dim, std::int64_t n0, int min_depth, void** out) {
  return guard([&] { *out = new Tree(build_tree(points(X, n, dim), n0, min_depth)); });
}
int orc_tree_depth(void* h) { return static_cast<Tree*>(h)->depth; }
std::int64_t orc_tree_level_size(void* h, int level) {
  return static_cast<std::int64_t>(static_cast<Tree*>(h)->levels[static_cast<size_t>(level)].size());
}
void orc_tree_perm(void* h, std::int64_t* out) {
  const Tree& t = *static_cast<Tree*>(h);
  std::memcpy(out, t.perm.data(), 8 * t.perm.size());
}
void orc_tree_level(void* h, int level, std::uint64_t* code, std::int64_t* begin, std::int64_t* end,
                    std::int64_t* parent, std::int64_t* nchild, std::int64_t* child8) {
  const auto& lv = static_cast<Tree*>(h)->levels[static_cast<size_t>(level)];
  for (size_t i = 0; i < lv.size(); ++i) {
    code[i] = lv[i].code;
    begin[i] = lv[i].begin;
    end[i] = lv[i].end;
    parent[i] = lv[i].parent;
    nchild[i] = lv[i].nchild;
    for (int c = 0; c < 8; ++c) child8[8 * i + c] = lv[i].child[c];
  }
}
void orc_tree_free(void* h) { delete static_cast<Tree*>(h); }

// Factorize with both trees built at a common depth (test helper make_trees).
int orc_factorize(const KernelDesc* kd, const double* X, std::int64_t nx, const double* Om, std::int64_t no,
                  int dim, std::int64_t n0, std::int64_t k, double eps, std::int64_t t, std::uint64_t seed,
                  int parallel, void** out) {
  return guard([&] {
    const MatXd XX = points(X, nx, dim), OO = points(Om, no, dim);
    auto tr = make_trees(XX, OO, n0);
    Config cfg;
    cfg.k_max = k;
    cfg.eps = eps;
    cfg.t = t;
    cfg.seed = seed;
    cfg.parallel = parallel != 0;
    *out = new Factorization(idbf_factorize(make_entry(*kd), tr.first, tr.second, XX, OO, cfg));
  });
}
// Factorize on explicitly given leaf sizes / depths (depth-mismatch pin).
int orc_factorize_trees(const KernelDesc* kd, const double* X, std::int64_t nx, const double* Om, std::int64_t no,
                        int dim, std::int64_t n0x, int mdx, std::int64_t n0o, int mdo, std::int64_t k, double eps,
                        std::int64_t t, std::uint64_t seed, void** out) {
  return guard([&] {
    const MatXd XX = points(X, nx, dim), OO = points(Om, no, dim);
    Tree tx = build_tree(XX, n0x, mdx), to = build_tree(OO, n0o, mdo);
    Config cfg;
    cfg.k_max = k;
    cfg.eps = eps;
    cfg.t = t;
    cfg.seed = seed;
    *out = new Factorization(idbf_factorize(make_entry(*kd), tx, to, XX, OO, cfg));
  });
}

// nrows ncols L h n0 nfactors total_nnz max_factor_nnz k_max t seed parallel
void orc_fac_info(void* h, std::int64_t* o) {
  const Factorization& F = *static_cast<Factorization*>(h);
  o[0] = F.nrows;
  o[1] = F.ncols;
  o[2] = F.L;
  o[3] = F.h;
  o[4] = F.n0;
  o[5] = static_cast<std::int64_t>(F.factors.size());
  o[6] = F.total_nnz();
  o[7] = F.max_factor_nnz();
  o[8] = F.cfg.k_max;
  o[9] = F.cfg.t;
  o[10] = static_cast<std::int64_t>(F.cfg.seed);
  o[11] = F.cfg.parallel ? 1 : 0;
}
double orc_fac_eps(void* h) { return static_cast<Factorization*>(h)->cfg.eps; }
double orc_fac_nnz_bound(void* h, double c) { return static_cast<Factorization*>(h)->nnz_bound(c); }
void orc_fac_perms(void* h, std::int64_t* rp, std::int64_t* cp) {
  const Factorization& F = *static_cast<Factorization*>(h);
  std::memcpy(rp, F.row_perm.data(), 8 * F.row_perm.size());
  std::memcpy(cp, F.col_perm.data(), 8 * F.col_perm.size());
}
// rows cols nblocks ngroups
void orc_fac_factor(void* h, int i, std::int64_t* o) {
  const Factor& f = static_cast<Factorization*>(h)->factors[static_cast<size_t>(i)];
  o[0] = f.rows;
  o[1] = f.cols;
  o[2] = static_cast<std::int64_t>(f.blocks.size());
  o[3] = static_cast<std::int64_t>(f.groups.size());
}
void orc_fac_tables(void* h, int i, std::int64_t* blocks4, std::int64_t* groups2) {
  const Factor& f = static_cast<Factorization*>(h)->factors[static_cast<size_t>(i)];
  for (size_t b = 0; b < f.blocks.size(); ++b) {
    blocks4[4 * b] = f.blocks[b].row_off;
    blocks4[4 * b + 1] = f.blocks[b].col_off;
    blocks4[4 * b + 2] = f.blocks[b].M.rows();
    blocks4[4 * b + 3] = f.blocks[b].M.cols();
  }
  for (size_t g = 0; g < f.groups.size(); ++g) {
    groups2[2 * g] = f.groups[g].first;
    groups2[2 * g + 1] = f.groups[g].second;
  }
}
void orc_fac_block(void* h, int i, std::int64_t b, double* out) {
  const Block& bl = static_cast<Factorization*>(h)->factors[static_cast<size_t>(i)].blocks[static_cast<size_t>(b)];
  std::memcpy(out, bl.M.d.data(), 16 * static_cast<size_t>(bl.M.size()));
}
void orc_fac_free(void* h) { delete static_cast<Factorization*>(h); }

int orc_apply(void* h, const double* in, std::int64_t in_len, std::int64_t nrhs, int tr, double* out, int parallel,
              int nthreads) {
  return guard([&] {
    const Factorization& F = *static_cast<Factorization*>(h);
    const Index nin = tr ? F.nrows : F.ncols;
    if (in_len != nin) throw std::invalid_argument("input length does not match the factorization");
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    apply(F, reinterpret_cast<const Cplx*>(in), nrhs, tr != 0, reinterpret_cast<Cplx*>(out), parallel != 0);
  });
}
int orc_save(void* h, const char* path) { return guard([&] { save(path, *static_cast<Factorization*>(h)); }); }
int orc_load(const char* path, void** out) { return guard([&] { *out = new Factorization(load(path)); }); }

int orc_direct_sum(const KernelDesc* kd, const double* f, const std::int64_t* rows, std::int64_t nrows, double* out,
                   int parallel, int nthreads) {
  return guard([&] {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    direct_sum(make_entry(*kd), kd->ncols, reinterpret_cast<const Cplx*>(f), rows, nrows,
               reinterpret_cast<Cplx*>(out), parallel != 0);
  });
}
int orc_entries(const KernelDesc* kd, const std::int64_t* ri, const std::int64_t* ci, std::int64_t n, double* out) {
  return guard([&] {
    EntryFn K = make_entry(*kd);
    for (std::int64_t q = 0; q < n; ++q) {
      const Cplx z = K(ri[q], ci[q]);
      out[2 * q] = z.real();
      out[2 * q + 1] = z.imag();
    }
  });
}
int orc_eps_b(const double* gb, std::int64_t N, const KernelDesc* kd, const double* f, std::int64_t n,
              std::int64_t nrows, std::uint64_t seed, double* out) {
  return guard([&] {
    *out = eps_b_of(reinterpret_cast<const Cplx*>(gb), N, make_entry(*kd), reinterpret_cast<const Cplx*>(f), n,
                    nrows, seed);
  });
}
void orc_random_coefficients(std::int64_t n, std::uint64_t seed, double* out) {
  random_coefficients(n, seed, reinterpret_cast<Cplx*>(out));
}
void orc_grid2d(std::int64_t n, double* X) { grid2d(n, X); }
double orc_fio2d_phase(const double* x, const double* xi) { return fio2d_phase(x, xi); }
double orc_fio3d_phase(const double* x, const double* xi) { return fio3d_phase(x, xi); }

// ---- linear-algebra pins (tests/test_linalg.cpp)
int orc_pqr(const double* A, std::int64_t m, std::int64_t n, int is_complex, std::int64_t max_rank,
            std::int64_t* perm, double* R, double* Q, std::int64_t* rank) {
  return guard([&] {
    if (is_complex) {
      QR<Cplx> q = pivoted_qr<Cplx>(from_colmajor<Cplx>(A, m, n), max_rank);
      std::memcpy(perm, q.perm.data(), 8 * q.perm.size());
      std::memcpy(R, q.R.d.data(), 16 * q.R.d.size());
      std::memcpy(Q, q.Q.d.data(), 16 * q.Q.d.size());
      *rank = q.rank;
    } else {
      QR<double> q = pivoted_qr<double>(from_colmajor<double>(A, m, n), max_rank);
      std::memcpy(perm, q.perm.data(), 8 * q.perm.size());
      std::memcpy(R, q.R.d.data(), 8 * q.R.d.size());
      std::memcpy(Q, q.Q.d.data(), 8 * q.Q.d.size());
      *rank = q.rank;
    }
  });
}
std::int64_t orc_id_rank(const double* d, std::int64_t m, std::int64_t k_max, double eps) {
  return id_rank(std::vector<double>(d, d + m), k_max, eps);
}
// V is k x n column-major (caller sizes it min(m,n) x n).
int orc_cid(const double* blk, std::int64_t m, std::int64_t n, std::int64_t k_max, double eps, std::int64_t* skel,
            double* V, std::int64_t* rank) {
  return guard([&] {
    ColumnID c = cid_from_rows(from_colmajor<Cplx>(blk, m, n), k_max, eps);
    std::memcpy(skel, c.skeleton.data(), 8 * c.skeleton.size());
    std::memcpy(V, c.V.d.data(), 16 * c.V.d.size());
    *rank = c.rank;
  });
}
// W is m x k column-major.
int orc_rid(const double* blk, std::int64_t m, std::int64_t n, std::int64_t k_max, double eps, std::int64_t* skel,
            double* W, std::int64_t* rank) {
  return guard([&] {
    RowID r = rid_from_cols(from_colmajor<Cplx>(blk, m, n), k_max, eps);
    std::memcpy(skel, r.skeleton.data(), 8 * r.skeleton.size());
    std::memcpy(W, r.W.d.data(), 16 * r.W.d.size());
    *rank = r.rank;
  });
}
std::int64_t orc_mock_cheb_rows(const double* pts, std::int64_t n, std::int64_t s, std::int64_t* out) {
  IndexVec r = mock_chebyshev_rows(std::vector<double>(pts, pts + n), s);
  std::memcpy(out, r.data(), 8 * r.size());
  return static_cast<std::int64_t>(r.size());
}
std::int64_t orc_mock_cheb_points(const double* P, std::int64_t n, int dim, std::int64_t s, std::uint64_t seed,
                                  std::int64_t* out) {
  std::mt19937_64 rng(seed);
  IndexVec r = mock_chebyshev_points(points(P, n, dim), s, rng);
  std::memcpy(out, r.data(), 8 * r.size());
  return static_cast<std::int64_t>(r.size());
}
std::int64_t orc_rand_subset(std::int64_t n, std::int64_t k, std::uint64_t seed, std::int64_t* out) {
  std::mt19937_64 rng(seed);
  IndexVec r = rand_subset(n, k, rng);
  std::memcpy(out, r.data(), 8 * r.size());
  return static_cast<std::int64_t>(r.size());
}

// Several rand_subset draws in sequence from ONE std::mt19937_64(seed), as
// consecutive calls on one engine (low_rank_phase_factorization / rsvd /
// eps_K draw their index sets this way, src/phase_md.cpp:198-199,
// src/linalg.cpp:186-189, src/metrics.cpp:61-71).  Outputs concatenated.
std::int64_t orc_rand_subset_seq(std::uint64_t seed, std::int64_t ndraw, const std::int64_t* ns,
                                 const std::int64_t* ks, std::int64_t* out) {
  std::mt19937_64 rng(seed);
  std::int64_t off = 0;
  for (std::int64_t d = 0; d < ndraw; ++d) {
    IndexVec r = rand_subset(ns[d], ks[d], rng);
    std::memcpy(out + off, r.data(), 8 * r.size());
    off += static_cast<std::int64_t>(r.size());
  }
  return off;
}

}  // extern "C"
