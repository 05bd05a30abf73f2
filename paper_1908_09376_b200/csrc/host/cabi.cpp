// C ABI over the host factorization object (include/midbf_b200.h, "host
// factorization object" section) plus the shared error plumbing.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>

#include "../status.hpp"
#include "midbf/butterfly_io.hpp"
#include "midbf_internal.hpp"

namespace midbf::detail {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

void rethrow(int rc) {
  if (rc == MIDBF_OK) return;
  const std::string msg = g_last_error;
  switch (rc) {
    case MIDBF_EINVAL:
      throw std::invalid_argument(msg);
    case MIDBF_ELOGIC:
      throw std::logic_error(msg);
    case MIDBF_ECUDA:
      throw CudaFailure(msg);
    default:
      throw std::runtime_error(msg);
  }
}

}  // namespace midbf::detail

using midbf::Index;
using midbf::detail::guard;

struct midbf_fact_s {
  midbf::bf::Factorization F;
  midbf::bf::FactorizeStats stats;
};

namespace {

midbf::MatXd points(const double* P, Index n, int dim) {
  midbf::MatXd M(n, dim);
  for (Index i = 0; i < n; ++i)
    for (int a = 0; a < dim; ++a) M(i, a) = P[i * dim + a];
  return M;
}

}  // namespace

extern "C" {

const char* midbf_last_error(void) { return midbf::detail::g_last_error.c_str(); }

uint64_t midbf_chain(uint64_t a, uint64_t b) {
  auto mix = [](uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
  };
  return mix(a ^ mix(b));
}

// src/experiment.cpp:75-81 (same libstdc++ distribution and call expression)
int midbf_random_coefficients(int64_t n, uint64_t seed, double* out) {
  return guard([&] {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> g(0.0, 1.0);
    auto* z = reinterpret_cast<midbf::Cplx*>(out);
    for (int64_t i = 0; i < n; ++i) z[i] = midbf::Cplx(g(rng), g(rng));
  });
}

int64_t midbf_rand_subset(int64_t n, int64_t k, uint64_t seed, int64_t* out) {
  std::mt19937_64 rng(seed);
  const midbf::IndexVec r = midbf::la::rand_subset(n, k, rng);
  std::memcpy(out, r.data(), 8 * r.size());
  return static_cast<int64_t>(r.size());
}

int midbf_factorize(midbf_fact_t* out, const midbf_kernel_desc* kernel, int64_t n0, int64_t k_max, double eps,
                    int64_t t, uint64_t seed, int exec, int sampler) {
  return guard([&] {
    if (!out || !kernel) throw std::invalid_argument("null argument");
    if (!kernel->X || !kernel->Omega || (kernel->dim != 2 && kernel->dim != 3))
      throw std::invalid_argument("factorize needs 2D/3D point sets X and Omega in the kernel description");
    static const bool timing = std::getenv("MIDBF_FACT_TIMING") != nullptr;
    const auto t_in = std::chrono::steady_clock::now();
    const midbf::MatXd X = points(kernel->X, kernel->nrows, kernel->dim);
    const midbf::MatXd O = points(kernel->Omega, kernel->ncols, kernel->dim);
    // both trees at a common depth (src/experiment.cpp:140-144)
    midbf::tree::ClusterTree tx, to;
    std::exception_ptr terr;
#pragma omp parallel sections num_threads(2)
    {
#pragma omp section
      {
        try {
          tx = midbf::tree::build_tree(X, n0);
        } catch (...) {
#pragma omp critical
          terr = std::current_exception();
        }
      }
#pragma omp section
      {
        try {
          to = midbf::tree::build_tree(O, n0);
        } catch (...) {
#pragma omp critical
          terr = std::current_exception();
        }
      }
    }
    if (terr) std::rethrow_exception(terr);
    const int L = std::max(tx.depth, to.depth);
    if (tx.depth != L) tx = midbf::tree::build_tree(X, n0, L);
    if (to.depth != L) to = midbf::tree::build_tree(O, n0, L);
    if (timing)
      std::fprintf(stderr, "[factorize] points + trees %.2f ms\n",
                   1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t_in).count());
    midbf::bf::Config cfg;
    cfg.rank = {k_max, eps};
    cfg.t = t;
    cfg.seed = seed;
    cfg.exec = exec ? midbf::Exec::Parallel : midbf::Exec::Serial;
    auto h = std::make_unique<midbf_fact_s>();
    if (sampler == 0 || sampler == 2) {
      h->F = midbf::bf::idbf_factorize_stats(*kernel, tx, to, X, O, cfg, &h->stats, sampler == 2);
    } else if (sampler == 1) {
      const midbf_kernel_desc kd = *kernel;
      midbf::bf::EntryFn K = [kd](Index i, Index j) { return midbf::ker::entry(kd, i, j); };
      h->F = midbf::bf::idbf_factorize(K, tx, to, X, O, cfg);
    } else {
      throw std::invalid_argument("sampler must be 0, 1 or 2");
    }
    if (timing)
      std::fprintf(stderr, "[factorize] total %.2f ms (library %.2f ms)\n",
                   1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t_in).count(),
                   1e3 * h->stats.seconds);
    *out = h.release();
  });
}

int midbf_fact_load(midbf_fact_t* out, const char* path) {
  return guard([&] {
    auto h = std::make_unique<midbf_fact_s>();
    h->F = midbf::bf::load_factorization(path);
    *out = h.release();
  });
}

int midbf_fact_save(midbf_fact_t fact, const char* path) {
  return guard([&] { midbf::bf::save_factorization(path, fact->F); });
}

int midbf_fact_destroy(midbf_fact_t fact) {
  return guard([&] { delete fact; });
}

int midbf_fact_info(midbf_fact_t fact, int64_t* o, double* eps) {
  return guard([&] {
    const auto& F = fact->F;
    o[0] = F.nrows;
    o[1] = F.ncols;
    o[2] = F.L;
    o[3] = F.h;
    o[4] = F.n0;
    o[5] = F.factor_count();
    o[6] = F.total_nnz();
    o[7] = F.max_factor_nnz();
    o[8] = F.cfg.rank.k_max;
    o[9] = F.cfg.t;
    o[10] = static_cast<int64_t>(F.cfg.seed);
    o[11] = F.cfg.exec == midbf::Exec::Parallel ? 1 : 0;
    if (eps) *eps = F.cfg.rank.eps;
  });
}

// Device-sampling statistics of the last factorize: entries, sampler calls.
int midbf_fact_stats(midbf_fact_t fact, int64_t* o) {
  return guard([&] {
    o[0] = fact->stats.entries;
    o[1] = fact->stats.launches;
    o[2] = static_cast<int64_t>(fact->stats.sample_seconds * 1e9);  // ns
  });
}

int midbf_fact_id_stats(midbf_fact_t fact, int64_t* o) {
  return guard([&] {
    o[0] = fact->stats.device_ids;
    o[1] = fact->stats.id_fallbacks;
    o[2] = static_cast<int64_t>(fact->stats.id_seconds * 1e9);  // ns
    o[3] = static_cast<int64_t>(fact->stats.seconds * 1e9);     // ns, whole factorization
  });
}

int midbf_fact_kernel_stats(midbf_fact_t fact, int64_t* o) {
  return guard([&] {
    o[0] = fact->stats.k3_launches;
    o[1] = fact->stats.k3_entries;
    o[2] = static_cast<int64_t>(fact->stats.k3_seconds * 1e9);  // ns
    o[3] = fact->stats.k5_launches;
    o[4] = static_cast<int64_t>(fact->stats.k5_seconds * 1e9);  // ns
  });
}

int midbf_fact_factor(midbf_fact_t fact, int64_t i, int64_t* o) {
  return guard([&] {
    if (i < 0 || i >= fact->F.factor_count()) throw std::invalid_argument("factor index out of range");
    const auto& f = fact->F.factors[static_cast<size_t>(i)];
    o[0] = f.rows;
    o[1] = f.cols;
    o[2] = static_cast<int64_t>(f.blocks.size());
    o[3] = static_cast<int64_t>(f.groups.size());
  });
}

int midbf_fact_tables(midbf_fact_t fact, int64_t i, int64_t* blocks4, int64_t* groups2) {
  return guard([&] {
    if (i < 0 || i >= fact->F.factor_count()) throw std::invalid_argument("factor index out of range");
    const auto& f = fact->F.factors[static_cast<size_t>(i)];
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
  });
}

int midbf_fact_block(midbf_fact_t fact, int64_t i, int64_t b, double* out) {
  return guard([&] {
    const auto& f = fact->F.factors.at(static_cast<size_t>(i));
    const auto& M = f.blocks.at(static_cast<size_t>(b)).M;
    std::memcpy(out, M.data(), static_cast<size_t>(16 * M.size()));
  });
}

int midbf_fact_perms(midbf_fact_t fact, int64_t* rp, int64_t* cp) {
  return guard([&] {
    std::memcpy(rp, fact->F.row_perm.data(), 8 * fact->F.row_perm.size());
    std::memcpy(cp, fact->F.col_perm.data(), 8 * fact->F.col_perm.size());
  });
}

int midbf_fact_plan(midbf_fact_t fact, unsigned directions, midbf_plan_t* out) {
  // both directions: a cache holding both is never rebuilt, so the returned
  // handle stays valid for the factorization's lifetime
  return guard([&] { *out = midbf::bf::device_plan(fact->F, directions | 3u)->plan; });
}

int midbf_fact_apply(midbf_fact_t fact, const double* f, double* g, int64_t nrhs, int transpose, void* stream) {
  return guard([&] {
    const auto cache = midbf::bf::device_plan(fact->F, transpose ? 2u : 1u);
    midbf::detail::rethrow(midbf_apply(cache->plan, f, g, nrhs, transpose, stream));
  });
}

}  // extern "C"
