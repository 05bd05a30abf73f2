// Scalar / dense-matrix aliases of the MIDBF host API.
//
// Replaces proj/include/midbf/types.hpp:11-22 of the reference, which aliases
// Eigen types.  Eigen is not part of this build: `Matrix<T>` is a small
// owning column-major container exposing the subset of the Eigen interface
// the factorize/apply API uses (rows(), cols(), size(), data(), operator()).
// Complex entries are std::complex<double> stored interleaved (re, im), the
// same bytes as Eigen::MatrixXcd and the MIDBF001 payload.
#pragma once

#include <complex>
#include <cstdint>
#include <vector>

namespace midbf {

using Index = std::int64_t;
using Cplx = std::complex<double>;
using IndexVec = std::vector<Index>;

template <class T>
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols) : r_(rows), c_(cols), d_(static_cast<size_t>(rows * cols)) {}
  static Matrix Zero(Index rows, Index cols) { return Matrix(rows, cols); }
  static Matrix Identity(Index rows, Index cols) {
    Matrix m(rows, cols);
    for (Index i = 0; i < rows && i < cols; ++i) m(i, i) = T(1);
    return m;
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  T* data() { return d_.data(); }
  const T* data() const { return d_.data(); }
  T& operator()(Index i, Index j) { return d_[static_cast<size_t>(i + j * r_)]; }
  const T& operator()(Index i, Index j) const { return d_[static_cast<size_t>(i + j * r_)]; }
  T& operator()(Index i) { return d_[static_cast<size_t>(i)]; }
  const T& operator()(Index i) const { return d_[static_cast<size_t>(i)]; }
  void resize(Index rows, Index cols) {
    r_ = rows;
    c_ = cols;
    d_.assign(static_cast<size_t>(rows * cols), T(0));
  }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<T> d_;
};

using MatXc = Matrix<Cplx>;
using MatXd = Matrix<double>;
using VecXc = Matrix<Cplx>;  // column vector: n x 1
using VecXd = Matrix<double>;

// Execution policy for host stages that also have a serial path
// (reference include/midbf/types.hpp:21-22).
enum class Exec { Serial, Parallel };

}  // namespace midbf
