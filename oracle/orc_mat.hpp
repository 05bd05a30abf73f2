// TEST INFRASTRUCTURE ONLY — part of the CPU oracle (see oracle/README.md).
// Minimal column-major dense matrix standing in for the Eigen aliases of the
// reference (proj/include/midbf/types.hpp:11-17).  Only what the restated
// hot path needs; no expression templates, sums run left to right.
#pragma once

#include <complex>
#include <cstdint>
#include <vector>

namespace orc {

using Index = std::int64_t;
using Cplx = std::complex<double>;
using IndexVec = std::vector<Index>;

template <class T>
struct Mat {
  Index r = 0, c = 0;
  std::vector<T> d;
  Mat() = default;
  Mat(Index rows, Index cols) : r(rows), c(cols), d(static_cast<size_t>(rows * cols)) {}
  T& operator()(Index i, Index j) { return d[static_cast<size_t>(i + j * r)]; }
  const T& operator()(Index i, Index j) const { return d[static_cast<size_t>(i + j * r)]; }
  T* col(Index j) { return d.data() + j * r; }
  const T* col(Index j) const { return d.data() + j * r; }
  Index size() const { return r * c; }
  Index rows() const { return r; }
  Index cols() const { return c; }
};

using MatXc = Mat<Cplx>;
using MatXd = Mat<double>;

inline double abs2(double x) { return x * x; }
inline double abs2(const Cplx& x) { return x.real() * x.real() + x.imag() * x.imag(); }
inline double conj_(double x) { return x; }
inline Cplx conj_(const Cplx& x) { return std::conj(x); }

}  // namespace orc
