// MIDBF001 container for the host Factorization (reference
// src/butterfly_io.cpp:63-167, layout include/midbf/butterfly_io.hpp:2-15),
// the kernel phase helpers (src/kernels.cpp:18-45, src/metrics.cpp:18-24),
// the device-plan cache and the sampled-row metric (src/metrics.cpp:26-53).
#include <cmath>
#include <cstring>
#include <mutex>
#include <fstream>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>

#include "../status.hpp"
#include "midbf/butterfly_io.hpp"
#include "midbf/metrics.hpp"
#include "midbf_internal.hpp"

namespace midbf {

namespace bf {

void save_factorization(const std::string& path, const Factorization& F) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open for writing: " + path);
  auto put = [&](const void* p) { f.write(static_cast<const char*>(p), 8); };
  auto i64 = [&](std::int64_t v) { put(&v); };
  f.write("MIDBF001", 8);
  for (std::int64_t v : {F.nrows, F.ncols, static_cast<std::int64_t>(F.L), static_cast<std::int64_t>(F.h), F.n0,
                         F.cfg.rank.k_max, F.cfg.t})
    i64(v);
  put(&F.cfg.rank.eps);
  const std::uint64_t seed = F.cfg.seed, ex = F.cfg.exec == Exec::Parallel ? 1u : 0u;
  put(&seed);
  put(&ex);
  i64(static_cast<std::int64_t>(F.factors.size()));
  f.write(reinterpret_cast<const char*>(F.row_perm.data()), static_cast<std::streamsize>(8 * F.row_perm.size()));
  f.write(reinterpret_cast<const char*>(F.col_perm.data()), static_cast<std::streamsize>(8 * F.col_perm.size()));
  for (const Factor& fc : F.factors) {
    for (std::int64_t v : {fc.rows, fc.cols, static_cast<std::int64_t>(fc.blocks.size()),
                           static_cast<std::int64_t>(fc.groups.size())})
      i64(v);
    for (const FactorBlock& b : fc.blocks)
      for (std::int64_t v : {b.row_off, b.col_off, b.M.rows(), b.M.cols()}) i64(v);
    for (const auto& g : fc.groups) {
      i64(g.first);
      i64(g.second);
    }
  }
  for (const Factor& fc : F.factors)
    for (const FactorBlock& b : fc.blocks)
      f.write(reinterpret_cast<const char*>(b.M.data()), static_cast<std::streamsize>(16 * b.M.size()));
  if (!f) throw std::runtime_error("short write to " + path);
}

Factorization load_factorization(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open for reading: " + path);
  auto need = [&](bool ok, const char* what) {
    if (!ok) throw std::runtime_error(std::string(what) + " in " + path);
  };
  auto word = [&]() {
    std::int64_t v = 0;
    f.read(reinterpret_cast<char*>(&v), 8);
    need(bool(f), "truncated container");
    return v;
  };
  const std::int64_t big = std::int64_t{1} << 40;
  auto count = [&](const char* what, std::int64_t mx) {
    const std::int64_t v = word();
    need(v >= 0 && v <= mx, what);
    return v;
  };
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
  F.cfg.rank.k_max = count("bad rank cap", big);
  F.cfg.t = count("bad sampling oversize", big);
  const std::int64_t e = word();
  std::memcpy(&F.cfg.rank.eps, &e, 8);
  F.cfg.seed = static_cast<std::uint64_t>(word());
  F.cfg.exec = word() ? Exec::Parallel : Exec::Serial;
  const std::int64_t nf = count("bad factor count", 4096);
  F.row_perm.resize(static_cast<size_t>(F.nrows));
  for (auto& v : F.row_perm) {
    v = count("bad row permutation entry", big);
    need(v < F.nrows, "row permutation out of range");
  }
  F.col_perm.resize(static_cast<size_t>(F.ncols));
  for (auto& v : F.col_perm) {
    v = count("bad column permutation entry", big);
    need(v < F.ncols, "column permutation out of range");
  }
  F.factors.resize(static_cast<size_t>(nf));
  for (Factor& fc : F.factors) {
    fc.rows = count("bad factor rows", big);
    fc.cols = count("bad factor cols", big);
    const std::int64_t nb = count("bad block count", big), ng = count("bad group count", big);
    fc.blocks.resize(static_cast<size_t>(nb));
    for (FactorBlock& b : fc.blocks) {
      b.row_off = count("bad block row offset", big);
      b.col_off = count("bad block column offset", big);
      const std::int64_t m = count("bad block height", big), n = count("bad block width", big);
      need(b.row_off + m <= fc.rows && b.col_off + n <= fc.cols, "block outside its factor");
      b.M.resize(m, n);
    }
    fc.groups.resize(static_cast<size_t>(ng));
    for (auto& g : fc.groups) {
      g.first = count("bad group begin", big);
      g.second = count("bad group end", big);
      need(g.first <= g.second && g.second <= nb, "group outside block table");
    }
  }
  for (Factor& fc : F.factors)
    for (FactorBlock& b : fc.blocks) {
      f.read(reinterpret_cast<char*>(b.M.data()), static_cast<std::streamsize>(16 * b.M.size()));
      need(bool(f), "truncated payload");
    }
  f.peek();
  need(f.eof(), "trailing bytes after payload");
  return F;
}

DevicePlanCache::~DevicePlanCache() {
  if (plan) midbf_plan_destroy(plan);
}

namespace {
// one mutex for all factorizations: plan builds are rare and brief
std::mutex& plan_cache_mutex() {
  static std::mutex mu;
  return mu;
}
// Layout stamp of a factorization: outer sizes, factor / block shapes and
// offsets, and the block buffers' addresses (a copied or reallocated block
// has a new buffer).  Cheap (no payload reads), so every apply checks it.
std::uint64_t layout_stamp(const Factorization& F) {
  std::uint64_t h = 0x6d69646266ull;
  auto mix = [&h](std::uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  };
  mix(static_cast<std::uint64_t>(F.nrows));
  mix(static_cast<std::uint64_t>(F.ncols));
  mix(F.row_perm.size());
  mix(F.col_perm.size());
  mix(reinterpret_cast<std::uintptr_t>(F.row_perm.data()));
  mix(reinterpret_cast<std::uintptr_t>(F.col_perm.data()));
  mix(F.factors.size());
  for (const Factor& fc : F.factors) {
    mix(static_cast<std::uint64_t>(fc.rows));
    mix(static_cast<std::uint64_t>(fc.cols));
    mix(fc.blocks.size());
    mix(fc.groups.size());
    for (const FactorBlock& b : fc.blocks) {
      mix(static_cast<std::uint64_t>(b.row_off));
      mix(static_cast<std::uint64_t>(b.col_off));
      mix(static_cast<std::uint64_t>(b.M.rows()));
      mix(static_cast<std::uint64_t>(b.M.cols()));
      mix(reinterpret_cast<std::uintptr_t>(b.M.data()));
    }
    for (const auto& g : fc.groups) {
      mix(static_cast<std::uint64_t>(g.first));
      mix(static_cast<std::uint64_t>(g.second));
    }
  }
  return h;
}
}  // namespace

void Factorization::invalidate_device_plan() const {
  std::lock_guard<std::mutex> lock(plan_cache_mutex());
  device.p.reset();  // callers holding the old cache keep it alive until they finish
}

std::shared_ptr<DevicePlanCache> device_plan(const Factorization& F, unsigned directions) {
  std::lock_guard<std::mutex> lock(plan_cache_mutex());
  const std::uint64_t stamp = layout_stamp(F);
  std::shared_ptr<DevicePlanCache>& cur = F.device.p;
  if (cur && cur->stamp != stamp) cur.reset();  // layout changed since the plan was built
  if (cur && (cur->directions & directions) == directions) return cur;
  const unsigned want = directions | (cur ? cur->directions : 0u);
  std::vector<std::int64_t> shape, blocks, groups;
  for (const Factor& fc : F.factors) {
    shape.insert(shape.end(), {fc.rows, fc.cols, static_cast<std::int64_t>(fc.blocks.size()),
                               static_cast<std::int64_t>(fc.groups.size())});
    for (const FactorBlock& b : fc.blocks) {
      blocks.insert(blocks.end(), {b.row_off, b.col_off, b.M.rows(), b.M.cols()});
    }
    for (const auto& g : fc.groups) groups.insert(groups.end(), {g.first, g.second});
  }
  std::vector<const double*> ptrs;  // per block, no repacking on the host
  ptrs.reserve(static_cast<size_t>(blocks.size() / 4));
  for (const Factor& fc : F.factors)
    for (const FactorBlock& b : fc.blocks) ptrs.push_back(reinterpret_cast<const double*>(b.M.data()));
  auto cache = std::make_shared<DevicePlanCache>();
  detail::rethrow(midbf_plan_create_blocks(&cache->plan, F.nrows, F.ncols, F.row_perm.data(), F.col_perm.data(),
                                           static_cast<std::int64_t>(F.factors.size()), shape.data(), blocks.data(),
                                           groups.data(), ptrs.data(), want));
  cache->directions = want;
  cache->stamp = stamp;
  cur = cache;  // earlier entries live on while callers still hold them
  return cache;
}

}  // namespace bf

namespace ker {

namespace {
const double kTwoPi = 6.283185307179586476925286766559;
}

double fio2d_phase(const double* x, const double* xi) {
  const double c1 = (2.0 + std::sin(kTwoPi * x[0]) * std::sin(kTwoPi * x[1])) / 16.0;
  const double c2 = (2.0 + std::cos(kTwoPi * x[0]) * std::cos(kTwoPi * x[1])) / 16.0;
  return x[0] * xi[0] + x[1] * xi[1] + std::sqrt(c1 * c1 * xi[0] * xi[0] + c2 * c2 * xi[1] * xi[1]);
}

double fio3d_phase(const double* x, const double* xi) {
  const double s0 = std::sin(kTwoPi * x[0]), s1 = std::sin(kTwoPi * x[1]), s2 = std::sin(kTwoPi * x[2]);
  const double c0 = std::cos(kTwoPi * x[0]), c1 = std::cos(kTwoPi * x[1]), c2 = std::cos(kTwoPi * x[2]);
  const double a1 = (2.0 + s0 * s1 * s2) / 16.0, a2 = (2.0 + c0 * c1 * c2) / 16.0, a3 = (2.0 + s0 * c1 * s2) / 16.0;
  return x[0] * xi[0] + x[1] * xi[1] + x[2] * xi[2] +
         std::sqrt(a1 * a1 * xi[0] * xi[0] + a2 * a2 * xi[1] * xi[1] + a3 * a3 * xi[2] * xi[2]);
}

MatXd grid2d(Index n) {
  MatXd X(n * n, 2);
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < n; ++j) {
      X(i * n + j, 0) = double(i) / double(n);
      X(i * n + j, 1) = double(j) / double(n);
    }
  return X;
}

Cplx entry(const KernelDesc& k, Index i, Index j) {
  switch (k.kind) {
    case MIDBF_KERNEL_FIO2D:
      return std::polar(1.0, kTwoPi * fio2d_phase(k.X + 2 * i, k.Omega + 2 * j));
    case MIDBF_KERNEL_FIO3D:
      return std::polar(1.0, kTwoPi * fio3d_phase(k.X + 3 * i, k.Omega + 3 * j));
    case MIDBF_KERNEL_LOWRANK: {
      double s = 0.0;
      for (int q = 0; q < k.rank; ++q) s += k.A[i * k.rank + q] * k.B[j * k.rank + q];
      return std::polar(1.0, kTwoPi * s);
    }
    case MIDBF_KERNEL_NUFFT: {
      double s = 0.0;
      for (int q = 0; q < k.dim; ++q) s += k.X[i * k.dim + q] * k.Omega[j * k.dim + q];
      return std::polar(1.0, kTwoPi * s);
    }
    case MIDBF_KERNEL_CONST:
      return {k.cre, k.cim};
    case MIDBF_KERNEL_RANK1:
      return Cplx(k.u[2 * i], k.u[2 * i + 1]) * Cplx(k.v[2 * j], k.v[2 * j + 1]);
    default:
      throw std::invalid_argument("unknown kernel kind");
  }
}

}  // namespace ker

namespace metrics {

double eps_b_of(const VecXc& g_b, const ker::KernelDesc& K, const VecXc& f, Index nrows, std::uint64_t seed) {
  const Index N = g_b.rows();
  if (nrows < 1) throw std::invalid_argument("eps_b: need at least one sampled row");
  std::mt19937_64 rng(seed);
  IndexVec S;
  if (nrows >= N) {
    S.resize(static_cast<size_t>(N));
    std::iota(S.begin(), S.end(), Index{0});
  } else {
    S = la::rand_subset(N, nrows, rng);
  }
  std::vector<Cplx> gd(S.size());
  detail::rethrow(midbf_direct_sum(&K, reinterpret_cast<const double*>(f.data()), S.data(),
                                   static_cast<std::int64_t>(S.size()), reinterpret_cast<double*>(gd.data())));
  double num = 0.0, den = 0.0;
  for (size_t q = 0; q < S.size(); ++q) {
    num += std::norm(g_b(S[q]) - gd[q]);
    den += std::norm(gd[q]);
  }
  return den == 0.0 ? std::sqrt(num) : std::sqrt(num / den);
}

double eps_b(const bf::Factorization& F, const ker::KernelDesc& K, const VecXc& f, Index nrows, std::uint64_t seed) {
  return eps_b_of(bf::apply(F, f), K, f, nrows, seed);
}

}  // namespace metrics

}  // namespace midbf
