// TEST INFRASTRUCTURE ONLY — a minimal stand-in for the Eigen3 API surface
// that the reference MIDBF sources use (/root/reference/proj/src/
// {butterfly,butterfly_io,linalg,tree,geometry,kernels,metrics,phase_md,
// phase1d}.cpp and the reference's own tests), so that those files compile
// UNMODIFIED in this image, where Eigen is absent.  The
// build (oracle/ref.mk) puts this directory first on the include path; the
// result lives only under oracle/_ref/ and is used only by tests/ to pin
// the oracle restatement (oracle/orc_core.cpp) and the product against the
// reference's own code.
//
// What this is NOT: Eigen.  Eigen3 is version-unpinned in the reference
// (proj/CMakeLists.txt:29) and its internal summation orders are not
// reproduced.  Arithmetic order here is the plain one, chosen to mirror the
// kinds of kernels Eigen dispatches to:
//   * y (+)= A * x with A column-major: axpy order (columns of A in order,
//     accumulated straight into y) — Eigen's col-major GEMV/GEMM;
//   * y (+)= A^T * x (a transposed / adjoint view): dot-product order (one
//     sequential inner product per output, then added) — Eigen's row-major GEMV;
//   * norms, squaredNorm, dot, sums: sequential from zero;
//   * triangular solves: back substitution, one right-hand side at a time;
//   * SVDs: one-sided Jacobi (accuracy ~1e-15 relative, not Eigen's digits).
// Everything is eager except views (blocks, rows, columns, transposes) and
// products, so the reference's `.noalias() +=` accumulations keep their
// order.
#pragma once

#include <algorithm>
#include <cassert>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstring>
#include <functional>
#include <initializer_list>
#include <limits>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
enum StorageOptions { ColMajor = 0, RowMajor = 1, AutoAlign = 0, DontAlign = 2 };
enum UpLoType { Lower = 1, Upper = 2, UnitLower = 5, UnitUpper = 6 };
enum DecompositionOptions { ComputeFullU = 4, ComputeThinU = 8, ComputeFullV = 16, ComputeThinV = 32 };

namespace shim {

template <class S>
struct real_of {
  using type = S;
};
template <class T>
struct real_of<std::complex<T>> {
  using type = T;
};
template <class S>
using real_t = typename real_of<S>::type;

template <class S>
struct is_cplx : std::false_type {};
template <class T>
struct is_cplx<std::complex<T>> : std::true_type {};

inline double cj(double x) { return x; }
inline float cj(float x) { return x; }
inline int cj(int x) { return x; }
inline long cj(long x) { return x; }
template <class T>
std::complex<T> cj(const std::complex<T>& z) {
  return std::conj(z);
}
inline double abs2(double x) { return x * x; }
template <class T>
T abs2(const std::complex<T>& z) {
  return z.real() * z.real() + z.imag() * z.imag();
}
inline double absv(double x) { return std::abs(x); }
template <class T>
T absv(const std::complex<T>& z) {
  return std::abs(z);
}

template <class A, class B>
struct promote {
  using type = decltype(std::declval<A>() * std::declval<B>());
};

struct DenseTag {};
template <class T>
constexpr bool is_dense_v = std::is_base_of_v<DenseTag, std::decay_t<T>>;

}  // namespace shim

template <class S, int R = Dynamic, int C = Dynamic, int O = 0, int MR = R, int MC = C>
class Matrix;
template <class S>
using PlainX = Matrix<S, Dynamic, Dynamic>;
template <class S>
class View;
template <class S>
class Product;
template <class S>
class NoAlias;
template <class S>
class DiagonalWrapper;
template <class S, int Mode>
class TriangularView;
template <class S>
class CommaInit;

// ---------------------------------------------------------------------------
// View: a strided window onto column-major storage (possibly conjugated).
// Copying a View copies the handle; ASSIGNING to a View writes its elements.
template <class S>
class View : public shim::DenseTag {
 public:
  using Scalar = S;
  using RealScalar = shim::real_t<S>;

  View() = default;
  View(S* p, Index r, Index c, Index rs, Index cs, bool conj = false)
      : p_(p), r_(r), c_(c), rs_(rs), cs_(cs), cj_(conj) {}
  View(const View&) = default;

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  Index innerStride() const { return rs_; }
  bool conjugated() const { return cj_; }
  Index outerStride() const { return cs_; }

  S coeff(Index i, Index j) const {
    const S v = p_[i * rs_ + j * cs_];
    return cj_ ? shim::cj(v) : v;
  }
  S& coeffRef(Index i, Index j) const { return p_[i * rs_ + j * cs_]; }
  S& operator()(Index i, Index j) const { return coeffRef(i, j); }
  // linear access: vectors along their length, matrices column-major
  S& lin(Index k) const {
    if (c_ == 1) return coeffRef(k, 0);
    if (r_ == 1) return coeffRef(0, k);
    return coeffRef(k % r_, k / r_);
  }
  S lincoeff(Index k) const {
    if (c_ == 1) return coeff(k, 0);
    if (r_ == 1) return coeff(0, k);
    return coeff(k % r_, k / r_);
  }
  S& operator()(Index k) const { return lin(k); }
  S& operator[](Index k) const { return lin(k); }
  S value() const { return coeff(0, 0); }

  // ---- sub-views
  View block(Index i, Index j, Index m, Index n) const {
    check_range(i, j, m, n);
    return View(p_ + i * rs_ + j * cs_, m, n, rs_, cs_, cj_);
  }
  View col(Index j) const { return block(0, j, r_, 1); }
  View row(Index i) const { return block(i, 0, 1, c_); }
  View middleRows(Index i, Index n) const { return block(i, 0, n, c_); }
  View middleCols(Index j, Index n) const { return block(0, j, r_, n); }
  View topRows(Index n) const { return block(0, 0, n, c_); }
  View bottomRows(Index n) const { return block(r_ - n, 0, n, c_); }
  View leftCols(Index n) const { return block(0, 0, r_, n); }
  View rightCols(Index n) const { return block(0, c_ - n, r_, n); }
  View topLeftCorner(Index m, Index n) const { return block(0, 0, m, n); }
  View topRightCorner(Index m, Index n) const { return block(0, c_ - n, m, n); }
  View bottomLeftCorner(Index m, Index n) const { return block(r_ - m, 0, m, n); }
  View bottomRightCorner(Index m, Index n) const { return block(r_ - m, c_ - n, m, n); }
  View head(Index n) const { return c_ == 1 ? block(0, 0, n, 1) : block(0, 0, 1, n); }
  View tail(Index n) const { return c_ == 1 ? block(r_ - n, 0, n, 1) : block(0, c_ - n, 1, n); }
  View segment(Index i, Index n) const { return c_ == 1 ? block(i, 0, n, 1) : block(0, i, 1, n); }
  View transpose() const { return View(p_, c_, r_, cs_, rs_, cj_); }
  View adjoint() const { return View(p_, c_, r_, cs_, rs_, shim::is_cplx<S>::value ? !cj_ : false); }
  PlainX<S> conjugate() const;
  PlainX<S> eval() const;

  // ---- reductions (sequential, from zero)
  RealScalar squaredNorm() const {
    RealScalar s = 0;
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) s += shim::abs2(coeff(i, j));
    return s;
  }
  RealScalar norm() const { return std::sqrt(squaredNorm()); }
  S sum() const {
    S s = S(0);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) s += coeff(i, j);
    return s;
  }
  S mean() const { return sum() / S(static_cast<RealScalar>(size())); }
  S prod() const {
    S s = S(1);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) s *= coeff(i, j);
    return s;
  }
  S trace() const {
    S s = S(0);
    for (Index i = 0; i < std::min(r_, c_); ++i) s += coeff(i, i);
    return s;
  }
  template <class T>
  auto dot(const View<T>& o) const {  // conjugate-linear in the first argument (Eigen's convention)
    using P = typename shim::promote<S, T>::type;
    if (size() != o.size()) throw std::invalid_argument("shim dot: size mismatch");
    P s = P(0);
    for (Index k = 0; k < size(); ++k) s += P(shim::cj(lincoeff(k))) * P(o.lincoeff(k));
    return s;
  }
  S minCoeff() const { return extreme(std::less<S>(), nullptr, nullptr); }
  S maxCoeff() const { return extreme(std::greater<S>(), nullptr, nullptr); }
  template <class I>
  S minCoeff(I* ri, I* ci = nullptr) const {
    Index a = 0, b = 0;
    const S v = extreme(std::less<S>(), &a, &b);
    set_index(ri, ci, a, b);
    return v;
  }
  template <class I>
  S maxCoeff(I* ri, I* ci = nullptr) const {
    Index a = 0, b = 0;
    const S v = extreme(std::greater<S>(), &a, &b);
    set_index(ri, ci, a, b);
    return v;
  }
  bool allFinite() const {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) {
        const S v = coeff(i, j);
        if (!std::isfinite(std::real(v)) || !std::isfinite(std::imag(v))) return false;
      }
    return true;
  }
  bool hasNaN() const {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) {
        const S v = coeff(i, j);
        if (std::isnan(std::real(v)) || std::isnan(std::imag(v))) return true;
      }
    return false;
  }
  Index count() const {
    Index n = 0;
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) n += coeff(i, j) != S(0);
    return n;
  }

  // ---- coefficient-wise (eager)
  PlainX<RealScalar> cwiseAbs() const;
  PlainX<RealScalar> cwiseAbs2() const;
  PlainX<RealScalar> real() const;
  PlainX<RealScalar> imag() const;
  PlainX<S> normalized() const;
  template <class F>
  PlainX<S> unaryExpr(F f) const;
  PlainX<S> cwiseProduct(const View& o) const;
  PlainX<S> cwiseQuotient(const View& o) const;
  PlainX<S> cwiseMax(const View& o) const;
  PlainX<S> cwiseMin(const View& o) const;
  template <class T>
  PlainX<T> cast() const;

  // ---- in place
  void normalize() const {
    const RealScalar n = norm();
    if (n > 0) *this /= S(n);
  }
  const View& setZero() const { return fill(S(0)); }
  const View& setOnes() const { return fill(S(1)); }
  const View& setConstant(const S& v) const { return fill(v); }
  const View& setIdentity() const {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) coeffRef(i, j) = i == j ? S(1) : S(0);
    return *this;
  }
  const View& fill(const S& v) const {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) coeffRef(i, j) = v;
    return *this;
  }
  void swap(const View& o) const {
    if (o.r_ != r_ || o.c_ != c_) throw std::invalid_argument("shim swap: size mismatch");
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) std::swap(coeffRef(i, j), o.coeffRef(i, j));
  }
  const View& operator*=(const S& a) const {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) coeffRef(i, j) *= a;
    return *this;
  }
  const View& operator/=(const S& a) const {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) coeffRef(i, j) /= a;
    return *this;
  }
  // assignment writes through (rhs evaluated first: no aliasing surprises)
  const View& operator=(const View& o) const {
    assign_from(PlainX<S>(o));
    return *this;
  }
  template <class E, class = std::enable_if_t<shim::is_dense_v<E>>>
  const View& operator=(const E& e) const {
    assign_from(PlainX<S>(e));
    return *this;
  }
  const View& operator=(const Product<S>& p) const;
  template <class E>
  const View& operator+=(const E& e) const;
  template <class E>
  const View& operator-=(const E& e) const;
  NoAlias<S> noalias() const;
  DiagonalWrapper<S> asDiagonal() const;
  template <int Mode>
  TriangularView<S, Mode> triangularView() const;
  CommaInit<S> operator<<(const S& v) const;

  S* data() const { return p_; }

 protected:
  void check_range(Index i, Index j, Index m, Index n) const {
    if (i < 0 || j < 0 || m < 0 || n < 0 || i + m > r_ || j + n > c_)
      throw std::out_of_range("shim block outside the matrix");
  }
  template <class Cmp>
  S extreme(Cmp cmp, Index* ri, Index* ci) const {
    if (size() == 0) throw std::invalid_argument("shim min/maxCoeff of an empty matrix");
    S best = coeff(0, 0);
    Index bi = 0, bj = 0;
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) {
        const S v = coeff(i, j);
        if (cmp(v, best)) {
          best = v;
          bi = i;
          bj = j;
        }
      }
    if (ri) *ri = bi;
    if (ci) *ci = bj;
    return best;
  }
  template <class I>
  void set_index(I* ri, I* ci, Index a, Index b) const {
    if (ci) {
      *ri = static_cast<I>(a);
      *ci = static_cast<I>(b);
    } else if (ri) {
      *ri = static_cast<I>(c_ == 1 ? a : (r_ == 1 ? b : a + b * r_));
    }
  }
  void assign_from(const PlainX<S>& src) const;

  S* p_ = nullptr;
  Index r_ = 0, c_ = 0, rs_ = 1, cs_ = 0;
  bool cj_ = false;
};

// ---------------------------------------------------------------------------
// Matrix: owning, column-major storage.  R / C only choose defaults (vector
// shapes, fixed sizes); every size is held at run time.
template <class S, int R, int C, int O, int MR, int MC>
class Matrix : public View<S> {
  using Base = View<S>;

 public:
  using Scalar = S;
  using RealScalar = shim::real_t<S>;
  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;

  Matrix() { init(R > 0 ? R : 0, C > 0 ? C : 0); }
  Matrix(const Matrix& o) : Base() { copy_from(o); }
  Matrix(Matrix&& o) noexcept : Base() { take(std::move(o)); }
  // one size argument: a vector of that length (or a fixed 1-vector value)
  template <class T, class = std::enable_if_t<std::is_integral_v<T>>>
  explicit Matrix(T n) {
    if (C == 1)
      init(static_cast<Index>(n), 1);
    else if (R == 1)
      init(1, static_cast<Index>(n));
    else
      init(static_cast<Index>(n), static_cast<Index>(n));
  }
  // two arguments: sizes, or the coefficients of a fixed 2-vector
  template <class A, class B, class = std::enable_if_t<std::is_arithmetic_v<A> && std::is_arithmetic_v<B>>>
  Matrix(A a, B b) {
    if constexpr (R * C == 2 && R > 0 && C > 0) {
      init(R, C);
      this->p_[0] = S(a);
      this->p_[1] = S(b);
    } else {
      init(static_cast<Index>(a), static_cast<Index>(b));
    }
  }
  Matrix(const S& a, const S& b, const S& c) {
    static_assert(R * C == 3, "three coefficients need a fixed 3-vector");
    init(R, C);
    this->p_[0] = a;
    this->p_[1] = b;
    this->p_[2] = c;
  }
  template <class E, class = std::enable_if_t<shim::is_dense_v<E>>>
  Matrix(const E& e) {
    from_view(e);
  }
  Matrix(const Product<S>& p);
  Matrix(const NoAlias<S>&) = delete;

  Matrix& operator=(const Matrix& o) {
    if (this != &o) {
      Matrix t(o);
      swap_storage(t);
    }
    return *this;
  }
  Matrix& operator=(Matrix&& o) noexcept {
    if (this != &o) take(std::move(o));
    return *this;
  }
  template <class E, class = std::enable_if_t<shim::is_dense_v<E>>>
  Matrix& operator=(const E& e) {
    Matrix t(e);
    swap_storage(t);
    return *this;
  }
  Matrix& operator=(const Product<S>& p) {
    Matrix t(p);
    swap_storage(t);
    return *this;
  }

  void resize(Index r, Index c) {
    if (r == this->r_ && c == this->c_) return;
    init(r, c);
  }
  void resize(Index n) {
    if (C == 1)
      resize(n, 1);
    else if (R == 1)
      resize(1, n);
    else
      throw std::invalid_argument("shim resize(n) on a matrix");
  }
  void conservativeResize(Index r, Index c) {
    Matrix t(r, c);
    for (Index j = 0; j < std::min(c, this->c_); ++j)
      for (Index i = 0; i < std::min(r, this->r_); ++i) t.p_[i + j * r] = this->p_[i + j * this->r_];
    swap_storage(t);
  }
  void conservativeResize(Index n) {
    if (C == 1)
      conservativeResize(n, 1);
    else
      conservativeResize(1, n);
  }
  Matrix& setZero() {
    Base::setZero();
    return *this;
  }
  Matrix& setZero(Index r, Index c) {
    resize(r, c);
    return setZero();
  }
  Matrix& setZero(Index n) {
    resize(n);
    return setZero();
  }
  Matrix& setOnes() {
    Base::setOnes();
    return *this;
  }
  Matrix& setConstant(Index r, Index c, const S& v) {
    resize(r, c);
    Base::fill(v);
    return *this;
  }
  Matrix& setIdentity() {
    Base::setIdentity();
    return *this;
  }
  Matrix& setIdentity(Index r, Index c) {
    resize(r, c);
    return setIdentity();
  }
  void swap(Matrix& o) { swap_storage(o); }
  void swap(Matrix&& o) { swap_storage(o); }
  using Base::swap;

  static Matrix Zero(Index r, Index c) {
    Matrix m(r, c);
    m.Base::setZero();
    return m;
  }
  static Matrix Zero(Index n) {
    Matrix m(n);
    m.Base::setZero();
    return m;
  }
  static Matrix Zero() {
    Matrix m;
    m.Base::setZero();
    return m;
  }
  static Matrix Ones(Index r, Index c) { return Constant(r, c, S(1)); }
  static Matrix Ones(Index n) {
    Matrix m(n);
    m.Base::fill(S(1));
    return m;
  }
  static Matrix Constant(Index r, Index c, const S& v) {
    Matrix m(r, c);
    m.Base::fill(v);
    return m;
  }
  static Matrix Constant(Index n, const S& v) {
    Matrix m(n);
    m.Base::fill(v);
    return m;
  }
  static Matrix Identity(Index r, Index c) {
    Matrix m(r, c);
    m.Base::setIdentity();
    return m;
  }
  static Matrix Identity(Index n) { return Identity(n, n); }
  static Matrix Identity() { return Identity(R, C); }
  static Matrix Unit(Index n, Index i) {
    Matrix m = Zero(n);
    m(i) = S(1);
    return m;
  }
  template <class F>
  static Matrix NullaryExpr(Index r, Index c, F f) {
    Matrix m(r, c);
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) m.p_[i + j * r] = f(i, j);
    return m;
  }
  template <class F>
  static Matrix NullaryExpr(Index n, F f) {
    Matrix m(n);
    for (Index i = 0; i < n; ++i) m.lin(i) = f(i);
    return m;
  }
  static Matrix LinSpaced(Index n, const S& lo, const S& hi) {
    Matrix m(n);
    for (Index i = 0; i < n; ++i) m.lin(i) = n == 1 ? hi : lo + (hi - lo) * S(i) / S(n - 1);
    return m;
  }

  S* data() { return this->p_; }
  const S* data() const { return this->p_; }

 private:
  void init(Index r, Index c) {
    if (r < 0 || c < 0) throw std::invalid_argument("shim matrix with a negative size");
    store_.assign(static_cast<size_t>(r * c), S(0));
    this->p_ = store_.data();
    this->r_ = r;
    this->c_ = c;
    this->rs_ = 1;
    this->cs_ = r;
    this->cj_ = false;
  }
  template <class E>
  void from_view(const E& e) {
    init(e.rows(), e.cols());
    for (Index j = 0; j < this->c_; ++j)
      for (Index i = 0; i < this->r_; ++i) this->p_[i + j * this->r_] = S(e.coeff(i, j));
  }
  void copy_from(const Matrix& o) {
    store_ = o.store_;
    this->p_ = store_.data();
    this->r_ = o.r_;
    this->c_ = o.c_;
    this->rs_ = 1;
    this->cs_ = o.r_;
    this->cj_ = false;
  }
  void take(Matrix&& o) {
    store_ = std::move(o.store_);
    this->p_ = store_.data();
    this->r_ = o.r_;
    this->c_ = o.c_;
    this->rs_ = 1;
    this->cs_ = o.r_;
    this->cj_ = false;
    o.store_.clear();
    o.p_ = nullptr;
    o.r_ = o.c_ = 0;
    o.cs_ = 0;
  }
  void swap_storage(Matrix& o) {
    std::swap(store_, o.store_);
    std::swap(this->r_, o.r_);
    std::swap(this->c_, o.c_);
    this->p_ = store_.data();
    o.p_ = o.store_.data();
    this->rs_ = o.rs_ = 1;
    this->cs_ = this->r_;
    o.cs_ = o.r_;
    this->cj_ = o.cj_ = false;
  }
  std::vector<S> store_;
};

template <class S>
PlainX<S> View<S>::eval() const {
  return PlainX<S>(*this);
}
template <class S>
PlainX<S> View<S>::conjugate() const {
  PlainX<S> m(*this);
  for (Index k = 0; k < m.size(); ++k) m.data()[k] = shim::cj(m.data()[k]);
  return m;
}
template <class S>
void View<S>::assign_from(const PlainX<S>& src) const {
  if (src.rows() != r_ || src.cols() != c_) {
    if (src.size() == size() && (r_ == 1 || c_ == 1) && (src.rows() == 1 || src.cols() == 1)) {
      for (Index k = 0; k < size(); ++k) lin(k) = src.lincoeff(k);  // vector of the other orientation
      return;
    }
    throw std::invalid_argument("shim assignment: size mismatch");
  }
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) coeffRef(i, j) = src.coeff(i, j);
}

#define MIDBF_SHIM_CWISE(NAME, TYPE, EXPR)            \
  template <class S>                                  \
  PlainX<shim::real_t<S>> View<S>::NAME() const {    \
    PlainX<shim::real_t<S>> m(r_, c_);                \
    for (Index j = 0; j < c_; ++j)                    \
      for (Index i = 0; i < r_; ++i) {                \
        const S v = coeff(i, j);                      \
        m(i, j) = EXPR;                               \
      }                                               \
    return m;                                         \
  }
MIDBF_SHIM_CWISE(cwiseAbs, RealScalar, shim::absv(v))
MIDBF_SHIM_CWISE(cwiseAbs2, RealScalar, shim::abs2(v))
MIDBF_SHIM_CWISE(real, RealScalar, std::real(v))
MIDBF_SHIM_CWISE(imag, RealScalar, std::imag(v))
#undef MIDBF_SHIM_CWISE

template <class S>
PlainX<S> View<S>::normalized() const {
  PlainX<S> m(*this);
  m.normalize();
  return m;
}
template <class S>
template <class F>
PlainX<S> View<S>::unaryExpr(F f) const {
  PlainX<S> m(r_, c_);
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) m(i, j) = f(coeff(i, j));
  return m;
}
template <class S>
PlainX<S> View<S>::cwiseProduct(const View& o) const {
  PlainX<S> m(r_, c_);
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) m(i, j) = coeff(i, j) * o.coeff(i, j);
  return m;
}
template <class S>
PlainX<S> View<S>::cwiseQuotient(const View& o) const {
  PlainX<S> m(r_, c_);
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) m(i, j) = coeff(i, j) / o.coeff(i, j);
  return m;
}
template <class S>
PlainX<S> View<S>::cwiseMax(const View& o) const {
  PlainX<S> m(r_, c_);
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) m(i, j) = std::max(coeff(i, j), o.coeff(i, j));
  return m;
}
template <class S>
PlainX<S> View<S>::cwiseMin(const View& o) const {
  PlainX<S> m(r_, c_);
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) m(i, j) = std::min(coeff(i, j), o.coeff(i, j));
  return m;
}
template <class S>
template <class T>
PlainX<T> View<S>::cast() const {
  PlainX<T> m(r_, c_);
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) m(i, j) = static_cast<T>(coeff(i, j));
  return m;
}

// ---------------------------------------------------------------------------
// Products.  A Product keeps views of its operands (and owns any operand
// that had to be materialised) until it is evaluated into a destination.
namespace shim {
// y (op)= a * b with the operand-layout-dependent order described at the top
template <class S>
void gemm_acc(const View<S>& y, const View<S>& a, const View<S>& b, bool subtract) {
  const Index m = a.rows(), k = a.cols(), n = b.cols();
  if (b.rows() != k || y.rows() != m || y.cols() != n) throw std::invalid_argument("shim product: size mismatch");
  // a transposed (row-major) view: dot-product order, then added
  const bool dot_order = a.rows() > 1 && a.innerStride() != 1;
  if (dot_order) {
    const bool raw = a.outerStride() == 1 && b.innerStride() == 1 && !a.conjugated() && !b.conjugated();
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < m; ++i) {
        S s = S(0);
        if constexpr (shim::is_cplx<S>::value) {
          if (raw) {  // a(i, :) and b(:, j) contiguous: same order, real arithmetic as above
            using T = typename S::value_type;
            const T* ad = reinterpret_cast<const T*>(&a.coeffRef(i, 0));
            const T* bd = reinterpret_cast<const T*>(&b.coeffRef(0, j));
            T sr = 0, si = 0;
            for (Index p = 0; p < k; ++p) {
              sr += ad[2 * p] * bd[2 * p] - ad[2 * p + 1] * bd[2 * p + 1];
              si += ad[2 * p] * bd[2 * p + 1] + ad[2 * p + 1] * bd[2 * p];
            }
            s = S(sr, si);
            if (subtract)
              y.coeffRef(i, j) -= s;
            else
              y.coeffRef(i, j) += s;
            continue;
          }
        }
        for (Index p = 0; p < k; ++p) s += a.coeff(i, p) * b.coeff(p, j);
        if (subtract)
          y.coeffRef(i, j) -= s;
        else
          y.coeffRef(i, j) += s;
      }
  } else {  // column-major: axpy order into y
    const bool raw = y.innerStride() == 1 && a.innerStride() == 1 && !a.conjugated();
    // output columns are independent: threads change no result bit
#pragma omp parallel for schedule(static) if (m * n * k > (1 << 20) && n > 1)
    for (Index j = 0; j < n; ++j)
      for (Index p = 0; p < k; ++p) {
        const S bpj = b.coeff(p, j);
        if (raw) {  // same order, contiguous columns
          S* yc = &y.coeffRef(0, j);
          const S* ac = &a.coeffRef(0, p);
          if constexpr (shim::is_cplx<S>::value) {
            // (a+bi)(c+di) = (ac - bd) + (ad + bc)i: the value std::complex's
            // product returns for finite operands (it only re-derives NaN
            // results), written out so the loop vectorises like Eigen's
            // packet kernels instead of calling __muldc3's slow path checks
            using T = typename S::value_type;
            T* yd = reinterpret_cast<T*>(yc);
            const T* ad = reinterpret_cast<const T*>(ac);
            const T c = bpj.real(), d = bpj.imag();
            if (subtract)
              for (Index i = 0; i < m; ++i) {
                const T re = ad[2 * i] * c - ad[2 * i + 1] * d, im = ad[2 * i] * d + ad[2 * i + 1] * c;
                yd[2 * i] -= re;
                yd[2 * i + 1] -= im;
              }
            else
              for (Index i = 0; i < m; ++i) {
                const T re = ad[2 * i] * c - ad[2 * i + 1] * d, im = ad[2 * i] * d + ad[2 * i + 1] * c;
                yd[2 * i] += re;
                yd[2 * i + 1] += im;
              }
          } else {
            if (subtract)
              for (Index i = 0; i < m; ++i) yc[i] -= ac[i] * bpj;
            else
              for (Index i = 0; i < m; ++i) yc[i] += ac[i] * bpj;
          }
          continue;
        }
        for (Index i = 0; i < m; ++i) {
          if (subtract)
            y.coeffRef(i, j) -= a.coeff(i, p) * bpj;
          else
            y.coeffRef(i, j) += a.coeff(i, p) * bpj;
        }
      }
  }
}
}  // namespace shim

template <class S>
class Product : public shim::DenseTag {
 public:
  using Scalar = S;
  Product(View<S> a, View<S> b, std::shared_ptr<PlainX<S>> ha, std::shared_ptr<PlainX<S>> hb)
      : a_(a), b_(b), ha_(std::move(ha)), hb_(std::move(hb)) {
    if (a_.cols() != b_.rows()) throw std::invalid_argument("shim product: inner dimensions differ");
  }
  Index rows() const { return a_.rows(); }
  Index cols() const { return b_.cols(); }
  Index size() const { return rows() * cols(); }
  void accumulate_into(const View<S>& y, bool subtract) const { shim::gemm_acc(y, a_, b_, subtract); }
  PlainX<S> eval() const {
    PlainX<S> y = PlainX<S>::Zero(rows(), cols());
    accumulate_into(y, false);
    return y;
  }
  S coeff(Index i, Index j) const { return eval().coeff(i, j); }
  // convenience (reductions / element access evaluate first)
  auto norm() const { return eval().norm(); }
  auto squaredNorm() const { return eval().squaredNorm(); }
  S operator()(Index i, Index j) const { return eval()(i, j); }
  S operator()(Index k) const { return eval()(k); }
  PlainX<S> transpose() const { return PlainX<S>(eval().transpose()); }
  PlainX<S> adjoint() const { return PlainX<S>(eval().adjoint()); }
  auto cwiseAbs() const { return eval().cwiseAbs(); }
  S value() const { return eval()(0, 0); }
  // an inner product (1 x 1) converts to its scalar, as in Eigen
  operator S() const {
    if (rows() != 1 || cols() != 1) throw std::invalid_argument("shim: only a 1x1 product converts to a scalar");
    return eval()(0, 0);
  }
  PlainX<S> col(Index j) const { return PlainX<S>(eval().col(j)); }
  PlainX<S> row(Index i) const { return PlainX<S>(eval().row(i)); }

 private:
  View<S> a_, b_;
  std::shared_ptr<PlainX<S>> ha_, hb_;
};

template <class S, int R, int C, int O, int MR, int MC>
Matrix<S, R, C, O, MR, MC>::Matrix(const Product<S>& p) {
  init(p.rows(), p.cols());
  p.accumulate_into(*this, false);
}

template <class S>
const View<S>& View<S>::operator=(const Product<S>& p) const {
  assign_from(p.eval());
  return *this;
}

template <class S>
class NoAlias {
 public:
  explicit NoAlias(View<S> v) : v_(v) {}
  const View<S>& operator+=(const Product<S>& p) const {
    p.accumulate_into(v_, false);
    return v_;
  }
  const View<S>& operator-=(const Product<S>& p) const {
    p.accumulate_into(v_, true);
    return v_;
  }
  const View<S>& operator=(const Product<S>& p) const {
    v_.setZero();
    p.accumulate_into(v_, false);
    return v_;
  }
  template <class E>
  const View<S>& operator+=(const E& e) const {
    return v_ += e;
  }
  template <class E>
  const View<S>& operator-=(const E& e) const {
    return v_ -= e;
  }
  template <class E>
  const View<S>& operator=(const E& e) const {
    return v_ = e;
  }

 private:
  View<S> v_;
};
template <class S>
NoAlias<S> View<S>::noalias() const {
  return NoAlias<S>(*this);
}

// ---- operand plumbing: any dense thing -> View<P> (+ an owner when it had
// to be materialised or promoted to the product scalar P)
namespace shim {
template <class E>
using scalar_of = typename std::decay_t<E>::Scalar;
template <class E>
auto plain(const E& e) {
  if constexpr (std::is_same_v<std::decay_t<E>, Product<scalar_of<E>>>)
    return e.eval();
  else
    return PlainX<scalar_of<E>>(e);
}
template <class P, class E>
View<P> as_view(E&& e, std::shared_ptr<PlainX<P>>& hold) {
  using D = std::decay_t<E>;
  if constexpr (std::is_same_v<D, Product<P>>) {
    hold = std::make_shared<PlainX<P>>(e.eval());
    return View<P>(*hold);
  } else if constexpr (std::is_same_v<D, View<P>>) {  // a handle: keep it
    return View<P>(e);
  } else if constexpr (std::is_base_of_v<View<P>, D>) {  // an owning matrix
    if constexpr (std::is_lvalue_reference_v<E&&>) {
      return View<P>(e);
    } else {  // a temporary: the product keeps it alive
      hold = std::make_shared<PlainX<P>>(PlainX<P>(e));
      return View<P>(*hold);
    }
  } else {  // another scalar type (or a product of one): promote
    const auto ev = plain(e);
    hold = std::make_shared<PlainX<P>>(ev.rows(), ev.cols());
    for (Index j = 0; j < ev.cols(); ++j)
      for (Index i = 0; i < ev.rows(); ++i) (*hold)(i, j) = P(ev.coeff(i, j));
    return View<P>(*hold);
  }
}
}  // namespace shim

template <class A, class B, class = std::enable_if_t<shim::is_dense_v<A> && shim::is_dense_v<B>>>
auto operator*(A&& a, B&& b) {
  using P = typename shim::promote<shim::scalar_of<A>, shim::scalar_of<B>>::type;
  std::shared_ptr<PlainX<P>> ha, hb;
  View<P> va = shim::as_view<P>(std::forward<A>(a), ha);
  View<P> vb = shim::as_view<P>(std::forward<B>(b), hb);
  return Product<P>(va, vb, ha, hb);
}

// ---- element-wise binary ops (eager)
namespace shim {
template <class A, class B, class F>
auto cwise(const A& a, const B& b, F f) {
  using P = typename promote<scalar_of<A>, scalar_of<B>>::type;
  if (a.rows() != b.rows() || a.cols() != b.cols()) {
    if (a.size() == b.size() && (a.rows() == 1 || a.cols() == 1) && (b.rows() == 1 || b.cols() == 1)) {
      PlainX<P> m(a.rows(), a.cols());
      const PlainX<P> ea(a), eb(b);
      for (Index k = 0; k < a.size(); ++k) m.lin(k) = f(ea.lincoeff(k), eb.lincoeff(k));
      return m;
    }
    throw std::invalid_argument("shim element-wise op: size mismatch");
  }
  PlainX<P> m(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) m(i, j) = f(P(a.coeff(i, j)), P(b.coeff(i, j)));
  return m;
}
}  // namespace shim

template <class A, class B, class = std::enable_if_t<shim::is_dense_v<A> && shim::is_dense_v<B>>>
auto operator+(const A& a, const B& b) {
  return shim::cwise(shim::plain(a), shim::plain(b), [](auto x, auto y) { return x + y; });
}
template <class A, class B, class = std::enable_if_t<shim::is_dense_v<A> && shim::is_dense_v<B>>>
auto operator-(const A& a, const B& b) {
  return shim::cwise(shim::plain(a), shim::plain(b), [](auto x, auto y) { return x - y; });
}
template <class A, class B, class = std::enable_if_t<shim::is_dense_v<A> && shim::is_dense_v<B>>>
bool operator==(const A& a, const B& b) {  // exact, coefficient-wise (Eigen: cwiseEqual().all())
  const auto ea = shim::plain(a);
  const auto eb = shim::plain(b);
  if (ea.rows() != eb.rows() || ea.cols() != eb.cols()) return false;
  for (Index j = 0; j < ea.cols(); ++j)
    for (Index i = 0; i < ea.rows(); ++i)
      if (!(ea(i, j) == eb(i, j))) return false;
  return true;
}
template <class A, class B, class = std::enable_if_t<shim::is_dense_v<A> && shim::is_dense_v<B>>>
bool operator!=(const A& a, const B& b) {
  return !(a == b);
}
template <class A, class = std::enable_if_t<shim::is_dense_v<A>>>
auto operator-(const A& a) {
  auto m = shim::plain(a);
  for (Index k = 0; k < m.size(); ++k) m.data()[k] = -m.data()[k];
  return m;
}
template <class A, class T,
          class = std::enable_if_t<shim::is_dense_v<A> && (std::is_arithmetic_v<T> || shim::is_cplx<T>::value)>>
auto operator*(const A& a, const T& s) {
  using P = typename shim::promote<shim::scalar_of<A>, T>::type;
  auto e = shim::plain(a);
  PlainX<P> m(e.rows(), e.cols());
  for (Index k = 0; k < m.size(); ++k) m.data()[k] = P(e.data()[k]) * P(s);
  return m;
}
template <class A, class T,
          class = std::enable_if_t<shim::is_dense_v<A> && (std::is_arithmetic_v<T> || shim::is_cplx<T>::value)>>
auto operator*(const T& s, const A& a) {
  using P = typename shim::promote<shim::scalar_of<A>, T>::type;
  auto e = shim::plain(a);
  PlainX<P> m(e.rows(), e.cols());
  for (Index k = 0; k < m.size(); ++k) m.data()[k] = P(s) * P(e.data()[k]);
  return m;
}
template <class A, class T,
          class = std::enable_if_t<shim::is_dense_v<A> && (std::is_arithmetic_v<T> || shim::is_cplx<T>::value)>>
auto operator/(const A& a, const T& s) {
  using P = typename shim::promote<shim::scalar_of<A>, T>::type;
  auto e = shim::plain(a);
  PlainX<P> m(e.rows(), e.cols());
  for (Index k = 0; k < m.size(); ++k) m.data()[k] = P(e.data()[k]) / P(s);
  return m;
}

template <class S>
template <class E>
const View<S>& View<S>::operator+=(const E& e) const {
  if constexpr (std::is_same_v<std::decay_t<E>, Product<S>>) {
    assign_from(PlainX<S>(*this + e.eval()));
  } else {
    const PlainX<S> t = *this + e;
    assign_from(t);
  }
  return *this;
}
template <class S>
template <class E>
const View<S>& View<S>::operator-=(const E& e) const {
  if constexpr (std::is_same_v<std::decay_t<E>, Product<S>>) {
    assign_from(PlainX<S>(*this - e.eval()));
  } else {
    const PlainX<S> t = *this - e;
    assign_from(t);
  }
  return *this;
}

// ---- diagonal matrices
template <class S>
class DiagonalWrapper {
 public:
  explicit DiagonalWrapper(PlainX<S> d) : d_(std::move(d)) {}
  const PlainX<S>& diagonal() const { return d_; }
  Index rows() const { return d_.size(); }
  Index cols() const { return d_.size(); }

 private:
  PlainX<S> d_;
};
template <class S>
DiagonalWrapper<S> View<S>::asDiagonal() const {
  return DiagonalWrapper<S>(PlainX<S>(*this));
}
template <class A, class T, class = std::enable_if_t<shim::is_dense_v<A>>>
auto operator*(const A& a, const DiagonalWrapper<T>& d) {
  using P = typename shim::promote<shim::scalar_of<A>, T>::type;
  auto e = shim::plain(a);
  PlainX<P> m(e.rows(), e.cols());
  for (Index j = 0; j < e.cols(); ++j)
    for (Index i = 0; i < e.rows(); ++i) m(i, j) = P(e(i, j)) * P(d.diagonal().lincoeff(j));
  return m;
}
template <class A, class T, class = std::enable_if_t<shim::is_dense_v<A>>>
auto operator*(const DiagonalWrapper<T>& d, const A& a) {
  using P = typename shim::promote<shim::scalar_of<A>, T>::type;
  auto e = shim::plain(a);
  PlainX<P> m(e.rows(), e.cols());
  for (Index j = 0; j < e.cols(); ++j)
    for (Index i = 0; i < e.rows(); ++i) m(i, j) = P(d.diagonal().lincoeff(i)) * P(e(i, j));
  return m;
}

// ---- triangular views (solve by substitution, one right-hand side at a time)
template <class S, int Mode>
class TriangularView {
 public:
  explicit TriangularView(View<S> a) : a_(a) {}
  template <class E>
  PlainX<S> solve(const E& rhs) const {
    PlainX<S> X(shim::plain(rhs));
    const Index n = a_.rows();
    if (a_.cols() != n || X.rows() != n) throw std::invalid_argument("shim triangular solve: size mismatch");
    const bool unit = (Mode & 4) != 0;
    for (Index j = 0; j < X.cols(); ++j) {
      if ((Mode & Upper) == Upper) {
        for (Index i = n - 1; i >= 0; --i) {
          S s = X(i, j);
          for (Index l = i + 1; l < n; ++l) s -= a_.coeff(i, l) * X(l, j);
          X(i, j) = unit ? s : s / a_.coeff(i, i);
        }
      } else {
        for (Index i = 0; i < n; ++i) {
          S s = X(i, j);
          for (Index l = 0; l < i; ++l) s -= a_.coeff(i, l) * X(l, j);
          X(i, j) = unit ? s : s / a_.coeff(i, i);
        }
      }
    }
    return X;
  }
  PlainX<S> toDenseMatrix() const {
    PlainX<S> m = PlainX<S>::Zero(a_.rows(), a_.cols());
    for (Index j = 0; j < a_.cols(); ++j)
      for (Index i = 0; i < a_.rows(); ++i)
        if (((Mode & Upper) == Upper && i <= j) || ((Mode & Lower) == Lower && i >= j)) m(i, j) = a_.coeff(i, j);
    return m;
  }

 private:
  View<S> a_;
};
template <class S>
template <int Mode>
TriangularView<S, Mode> View<S>::triangularView() const {
  return TriangularView<S, Mode>(*this);
}

// ---- comma initializer (row-major fill, as Eigen's <<)
template <class S>
class CommaInit {
 public:
  CommaInit(View<S> v, const S& first) : v_(v) { push(first); }
  CommaInit& operator,(const S& x) {
    push(x);
    return *this;
  }
  ~CommaInit() noexcept(false) {
    if (k_ != v_.size() && !std::uncaught_exceptions()) throw std::invalid_argument("shim comma initializer: too few coefficients");
  }

 private:
  void push(const S& x) {
    if (k_ >= v_.size()) throw std::invalid_argument("shim comma initializer: too many coefficients");
    const Index i = k_ / v_.cols(), j = k_ % v_.cols();
    v_(i, j) = x;
    ++k_;
  }
  View<S> v_;
  Index k_ = 0;
};
template <class S>
CommaInit<S> View<S>::operator<<(const S& v) const {
  return CommaInit<S>(*this, v);
}

// ---- Ref: a read-only parameter type (holds a copy; enough for const Ref)
template <class PlainT, int Options = 0, class StrideT = void>
class Ref : public std::remove_const_t<PlainT> {
  using Base = std::remove_const_t<PlainT>;

 public:
  template <class E, class = std::enable_if_t<shim::is_dense_v<E>>>
  Ref(const E& e) : Base(e) {}
};

// ---------------------------------------------------------------------------
// Householder QR (unpivoted) with a lazily applied Q
template <class S>
class HouseholderSequence {
 public:
  HouseholderSequence(std::shared_ptr<const PlainX<S>> qr, std::vector<S> tau) : qr_(std::move(qr)), tau_(std::move(tau)) {}
  template <class E>
  PlainX<S> operator*(const E& rhs) const {
    PlainX<S> B(shim::plain(rhs));
    const Index m = qr_->rows();
    if (B.rows() != m) throw std::invalid_argument("shim householderQ product: size mismatch");
    for (Index k = static_cast<Index>(tau_.size()) - 1; k >= 0; --k) apply_h(k, B);
    return B;
  }
  operator PlainX<S>() const { return *this * PlainX<S>::Identity(qr_->rows(), qr_->rows()); }

 private:
  void apply_h(Index k, PlainX<S>& B) const {  // B <- P_k^H B, v = [1; qr(k+1:, k)]
    const Index m = qr_->rows();
    for (Index j = 0; j < B.cols(); ++j) {
      S w = B(k, j);
      for (Index i = k + 1; i < m; ++i) w += shim::cj((*qr_)(i, k)) * B(i, j);
      w *= shim::cj(tau_[static_cast<size_t>(k)]);  // Q = P_0^H P_1^H ..., P_k = I - tau_k v v^H
      B(k, j) -= w;
      for (Index i = k + 1; i < m; ++i) B(i, j) -= (*qr_)(i, k) * w;
    }
  }
  std::shared_ptr<const PlainX<S>> qr_;
  std::vector<S> tau_;
};

template <class M>
class HouseholderQR {
  using S = typename M::Scalar;

 public:
  HouseholderQR() = default;
  template <class E>
  explicit HouseholderQR(const E& a) {
    compute(a);
  }
  template <class E>
  HouseholderQR& compute(const E& a) {
    auto A = std::make_shared<PlainX<S>>(shim::plain(a));
    const Index m = A->rows(), n = A->cols(), steps = std::min(m, n);
    tau_.assign(static_cast<size_t>(steps), S(0));
    for (Index k = 0; k < steps; ++k) {
      shim::real_t<S> tail2 = 0;
      for (Index i = k + 1; i < m; ++i) tail2 += shim::abs2((*A)(i, k));
      const S a0 = (*A)(k, k);
      if (tail2 == 0 && std::imag(a0) == 0) {
        tau_[static_cast<size_t>(k)] = S(0);
        continue;
      }
      const shim::real_t<S> xn = std::sqrt(shim::abs2(a0) + tail2);
      const shim::real_t<S> beta = std::real(a0) >= 0 ? -xn : xn;
      const S v0 = a0 - S(beta);
      for (Index i = k + 1; i < m; ++i) (*A)(i, k) /= v0;
      tau_[static_cast<size_t>(k)] = shim::cj((S(beta) - a0) / S(beta));
      (*A)(k, k) = S(beta);
      for (Index j = k + 1; j < n; ++j) {  // A(k:, j) <- H^H A(k:, j)
        S w = (*A)(k, j);
        for (Index i = k + 1; i < m; ++i) w += shim::cj((*A)(i, k)) * (*A)(i, j);
        w *= tau_[static_cast<size_t>(k)];
        (*A)(k, j) -= w;
        for (Index i = k + 1; i < m; ++i) (*A)(i, j) -= (*A)(i, k) * w;
      }
    }
    qr_ = A;
    return *this;
  }
  HouseholderSequence<S> householderQ() const { return HouseholderSequence<S>(qr_, tau_); }
  const PlainX<S>& matrixQR() const { return *qr_; }

 private:
  std::shared_ptr<const PlainX<S>> qr_;
  std::vector<S> tau_;
};

// ---------------------------------------------------------------------------
// SVD by one-sided Jacobi (Hestenes) on the taller orientation.  Singular
// values descending; thin U / V on request.
template <class M, int QRPreconditioner = 0>
class JacobiSVD {
  using S = typename M::Scalar;
  using Rl = shim::real_t<S>;

 public:
  JacobiSVD() = default;
  template <class E>
  explicit JacobiSVD(const E& a, unsigned opts = 0) {
    compute(a, opts);
  }
  template <class E>
  JacobiSVD& compute(const E& a, unsigned opts = 0) {
    PlainX<S> A(shim::plain(a));
    const bool flip = A.rows() < A.cols();
    PlainX<S> W0 = flip ? PlainX<S>(A.adjoint()) : A;  // m >= n
    const Index m = W0.rows(), n = W0.cols();
    // tall input: Householder QR first, Jacobi on the n x n R factor
    const bool pre = m > n;
    HouseholderQR<PlainX<S>> qr;
    PlainX<S> W;
    if (pre) {
      qr.compute(W0);
      W = PlainX<S>::Zero(n, n);
      for (Index j = 0; j < n; ++j)
        for (Index i = 0; i <= j; ++i) W(i, j) = qr.matrixQR()(i, j);
    } else {
      W = W0;
    }
    const Index mw = W.rows();
    PlainX<S> V = PlainX<S>::Identity(n, n);
    for (int sweep = 0; sweep < 80; ++sweep) {
      bool rotated = false;
      for (Index p = 0; p + 1 < n; ++p)
        for (Index q = p + 1; q < n; ++q) {
          S* wp = W.data() + p * mw;
          S* wq = W.data() + q * mw;
          Rl app = 0, aqq = 0;
          S apq = S(0);
          for (Index i = 0; i < mw; ++i) {
            app += shim::abs2(wp[i]);
            aqq += shim::abs2(wq[i]);
            apq += shim::cj(wp[i]) * wq[i];
          }
          const Rl g = std::abs(apq);
          if (g == 0 || g <= std::numeric_limits<Rl>::epsilon() * std::sqrt(app * aqq)) continue;
          rotated = true;
          // rotate columns p, q so that they become orthogonal
          const S ph = apq / g;  // unit phase
          const Rl zeta = (aqq - app) / (2 * g);
          const Rl t = (zeta >= 0 ? 1 : -1) / (std::abs(zeta) + std::sqrt(1 + zeta * zeta));
          const Rl c = 1 / std::sqrt(1 + t * t), sn = c * t;
          const S a12 = S(sn) * shim::cj(ph), a21 = S(sn) * ph;
          for (Index i = 0; i < mw; ++i) {
            const S x = wp[i], y = wq[i];
            wp[i] = S(c) * x - a12 * y;
            wq[i] = a21 * x + S(c) * y;
          }
          S* vp = V.data() + p * n;
          S* vq = V.data() + q * n;
          for (Index i = 0; i < n; ++i) {
            const S x = vp[i], y = vq[i];
            vp[i] = S(c) * x - a12 * y;
            vq[i] = a21 * x + S(c) * y;
          }
        }
      if (!rotated) break;
    }
    std::vector<Rl> sv(static_cast<size_t>(n));
    for (Index j = 0; j < n; ++j) sv[static_cast<size_t>(j)] = W.col(j).norm();
    std::vector<Index> ord(static_cast<size_t>(n));
    std::iota(ord.begin(), ord.end(), Index{0});
    std::stable_sort(ord.begin(), ord.end(), [&](Index x, Index y) { return sv[size_t(x)] > sv[size_t(y)]; });
    sing_.resize(n, 1);
    PlainX<S> U(mw, n), Vs(n, n);
    for (Index k = 0; k < n; ++k) {
      const Index j = ord[static_cast<size_t>(k)];
      sing_(k) = sv[static_cast<size_t>(j)];
      for (Index i = 0; i < n; ++i) Vs(i, k) = V(i, j);
      for (Index i = 0; i < mw; ++i) U(i, k) = sing_(k) > 0 ? W(i, j) / S(sing_(k)) : S(0);
    }
    complete(U, sing_);
    if (pre) {  // U = Q [U_R; 0]
      PlainX<S> Ur = PlainX<S>::Zero(m, n);
      for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) Ur(i, j) = U(i, j);
      U = qr.householderQ() * Ur;
    }
    if (!flip) {
      u_ = U;
      v_ = Vs;
    } else {  // A^H = U S V^H  =>  A = V S U^H
      u_ = Vs;
      v_ = U;
    }
    (void)opts;
    return *this;
  }
  const Matrix<Rl, Dynamic, 1>& singularValues() const { return sing_; }
  const PlainX<S>& matrixU() const { return u_; }
  const PlainX<S>& matrixV() const { return v_; }
  Index rank() const {
    Index r = 0;
    const Rl tol = sing_.size() ? sing_(0) * std::numeric_limits<Rl>::epsilon() * std::max(u_.rows(), v_.rows()) : 0;
    for (Index k = 0; k < sing_.size(); ++k) r += sing_(k) > tol;
    return r;
  }

 private:
  // columns of zero singular values: an orthonormal completion
  static void complete(PlainX<S>& U, const Matrix<Rl, Dynamic, 1>& s) {
    const Index m = U.rows();
    for (Index k = 0; k < U.cols(); ++k) {
      if (s(k) > 0) continue;
      for (Index e = 0; e < m; ++e) {
        PlainX<S> v = PlainX<S>::Zero(m, 1);
        v(e, 0) = S(1);
        for (Index q = 0; q < U.cols(); ++q) {
          if (q == k || (s(q) <= 0 && q > k)) continue;
          S d = S(0);
          for (Index i = 0; i < m; ++i) d += shim::cj(U(i, q)) * v(i, 0);
          for (Index i = 0; i < m; ++i) v(i, 0) -= d * U(i, q);
        }
        const Rl nv = v.norm();
        if (nv > 0.5) {
          for (Index i = 0; i < m; ++i) U(i, k) = v(i, 0) / S(nv);
          break;
        }
      }
    }
  }
  Matrix<Rl, Dynamic, 1> sing_;
  PlainX<S> u_, v_;
};
template <class M>
using BDCSVD = JacobiSVD<M>;

// ---------------------------------------------------------------------------
// Geometry: AngleAxis (Rodrigues)
template <class T>
class AngleAxis {
 public:
  template <class E>
  AngleAxis(T angle, const E& axis) : a_(angle), ax_(shim::plain(axis)) {}
  Matrix<T, 3, 3> toRotationMatrix() const {
    const T c = std::cos(a_), s = std::sin(a_), x = ax_.lincoeff(0), y = ax_.lincoeff(1), z = ax_.lincoeff(2);
    Matrix<T, 3, 3> R;
    R(0, 0) = c + x * x * (1 - c);
    R(0, 1) = x * y * (1 - c) - z * s;
    R(0, 2) = x * z * (1 - c) + y * s;
    R(1, 0) = y * x * (1 - c) + z * s;
    R(1, 1) = c + y * y * (1 - c);
    R(1, 2) = y * z * (1 - c) - x * s;
    R(2, 0) = z * x * (1 - c) - y * s;
    R(2, 1) = z * y * (1 - c) + x * s;
    R(2, 2) = c + z * z * (1 - c);
    return R;
  }

 private:
  T a_;
  PlainX<T> ax_;
};
using AngleAxisd = AngleAxis<double>;

// ---------------------------------------------------------------------------
// the usual typedefs
template <class S, int N = Dynamic>
using Vector = Matrix<S, N, 1>;
template <class S, int N = Dynamic>
using RowVector = Matrix<S, 1, N>;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using MatrixXcd = Matrix<std::complex<double>, Dynamic, Dynamic>;
using MatrixXi = Matrix<int, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using VectorXcd = Matrix<std::complex<double>, Dynamic, 1>;
using VectorXi = Matrix<int, Dynamic, 1>;
using RowVectorXd = Matrix<double, 1, Dynamic>;
using RowVectorXcd = Matrix<std::complex<double>, 1, Dynamic>;
using Matrix2d = Matrix<double, 2, 2>;
using Matrix3d = Matrix<double, 3, 3>;
using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using RowVector2d = Matrix<double, 1, 2>;
using RowVector3d = Matrix<double, 1, 3>;

}  // namespace Eigen
