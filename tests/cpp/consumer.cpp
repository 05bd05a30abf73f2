// A C++ consumer of the drop-in headers (include/midbf/*.hpp) linked
// against libmidbf_b200.so — what a user of the reference's C++ API
// (proj/include/midbf/butterfly.hpp:117-126, butterfly_io.hpp:24-28) compiles
// after switching.  Built by tests/test_cpp_consumer.py; run on a GPU.
//   1. bf::idbf_factorize with the reference's EntryFn callback (host entries)
//      and with a typed KernelDesc (GPU entries + IDs);
//   2. bf::apply / bf::apply_transpose (GPU) vs a dense direct product;
//   3. bf::save_factorization / load_factorization round trip, bitwise apply;
//   4. copy semantics of the device-plan cache: a copy edited after the
//      original was applied uses its own arenas; in-place edits need
//      invalidate_device_plan().
// Prints one line per check and exits non-zero on the first failure.
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <stdexcept>
#include <string>

#include "midbf/butterfly.hpp"
#include "midbf/butterfly_io.hpp"
#include "midbf/kernels.hpp"
#include "midbf/tree.hpp"

using namespace midbf;

namespace {
constexpr double kTwoPi = 6.283185307179586476925286766559;

void need(bool ok, const std::string& what) {
  std::printf("%s %s\n", ok ? "ok  " : "FAIL", what.c_str());
  if (!ok) std::exit(1);
}

double rel(const MatXc& a, const MatXc& b) {
  double num = 0, den = 0;
  for (Index i = 0; i < a.size(); ++i) {
    num += std::norm(a(i) - b(i));
    den += std::norm(b(i));
  }
  return std::sqrt(num / den);
}

bool same(const MatXc& a, const MatXc& b) {
  if (a.size() != b.size()) return false;
  for (Index i = 0; i < a.size(); ++i)
    if (a(i) != b(i)) return false;
  return true;
}
}  // namespace

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/tmp";
  const Index n = 32, N = n * n;
  const MatXd X = ker::grid2d(n);  // xi = x, the reference tests' setting
  tree::ClusterTree tx = tree::build_tree(X, 64), to = tree::build_tree(X, 64);
  need(tx.depth == 2 && to.depth == 2, "build_tree depth 2 at n=32, n0=64");

  bf::EntryFn K = [&X](Index i, Index j) {  // src/kernels.cpp:242-245
    const double x[2] = {X(i, 0), X(i, 1)}, xi[2] = {X(j, 0), X(j, 1)};
    return std::polar(1.0, kTwoPi * ker::fio2d_phase(x, xi));
  };
  bf::Config cfg;
  cfg.rank = {30, 1e-9};
  cfg.exec = Exec::Parallel;
  bf::Factorization F = bf::idbf_factorize(K, tx, to, X, X, cfg);
  need(F.factor_count() == 5, "EntryFn factorization has 2(L-h+1)+1 = 5 factors");

  std::mt19937_64 rng(7);
  std::normal_distribution<double> g01(0.0, 1.0);
  MatXc f(N, 1), dense_g(N, 1), ft(N, 1), dense_gt(N, 1);
  for (Index i = 0; i < N; ++i) f(i) = Cplx(g01(rng), g01(rng));
  for (Index i = 0; i < N; ++i) ft(i) = Cplx(g01(rng), g01(rng));
  for (Index i = 0; i < N; ++i) {
    Cplx a(0, 0), b(0, 0);
    for (Index j = 0; j < N; ++j) {
      a += K(i, j) * f(j);
      b += K(j, i) * ft(j);
    }
    dense_g(i) = a;
    dense_gt(i) = b;
  }
  const MatXc g = bf::apply(F, f);
  need(rel(g, dense_g) <= 1e-5, "bf::apply vs dense K f <= 1e-5 (tests/test_butterfly.cpp:202)");
  const MatXc gt = bf::apply_transpose(F, ft);
  need(rel(gt, dense_gt) <= 1e-5, "bf::apply_transpose vs dense K^T g <= 1e-5 (:205)");
  bool threw = false;
  try {
    bf::apply(F, MatXc(N - 1, 1));
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  need(threw, "length mismatch throws std::invalid_argument (src/butterfly.cpp:645)");

  // the same factorization with every entry and ID on the GPU
  midbf_kernel_desc kd{};
  kd.kind = MIDBF_KERNEL_FIO2D;
  kd.dim = 2;
  kd.nrows = kd.ncols = N;
  std::vector<double> xr(2 * N);
  for (Index i = 0; i < N; ++i) {
    xr[2 * i] = X(i, 0);
    xr[2 * i + 1] = X(i, 1);
  }
  kd.X = kd.Omega = xr.data();
  const bf::Factorization Fd = bf::idbf_factorize(kd, tx, to, X, X, cfg);
  need(rel(bf::apply(Fd, f), dense_g) <= 1e-5, "KernelDesc (GPU-sampled) factorization vs dense <= 1e-5");

  const std::string path = dir + "/consumer_" + std::to_string(::getpid()) + ".midbf";
  bf::save_factorization(path, F);
  const bf::Factorization L = bf::load_factorization(path);
  std::remove(path.c_str());
  need(L.total_nnz() == F.total_nnz() && same(bf::apply(L, f), g), "save / load round trip: bitwise apply");

  // copies do not share device arenas
  bf::Factorization C = F;
  C.factors[0].blocks[0].M(0, 0) *= 2.0;
  const MatXc gc = bf::apply(C, f);
  need(!same(gc, g), "an edited copy applies its own factors");
  need(same(bf::apply(F, f), g), "the original is unaffected by the copy's edit");
  // in-place value edits need invalidate_device_plan()
  F.factors[0].blocks[0].M(0, 0) *= 2.0;
  F.invalidate_device_plan();
  need(same(bf::apply(F, f), gc), "invalidate_device_plan picks up in-place edits");
  // layout edits are detected without it
  F.factors[0].blocks.pop_back();
  F.factors[0].groups.back().second -= 1;
  if (F.factors[0].groups.back().second == F.factors[0].groups.back().first) F.factors[0].groups.pop_back();
  need(!same(bf::apply(F, f), gc), "a layout change rebuilds the cached plan");
  std::printf("consumer ok\n");
  return 0;
}
