// TEST INFRASTRUCTURE ONLY (oracle/_ref): a minimal, eagerly evaluated
// stand-in for the subset of the Eigen 3 dense API that the reference
// headers (/root/reference/proj/include/hdivmg/*.hpp) use, so that those
// UNMODIFIED headers compile and run here (Eigen 3 itself is absent from the
// image). Semantics follow Eigen's documented behaviour (column-major
// storage, Block views that write through, PartialPivLU / FullPivLU / LDLT /
// JacobiSVD solves); expressions are evaluated immediately instead of lazily,
// which changes nothing but aliasing corner cases the reference does not hit.
// Arithmetic order is the plain sequential one (no SIMD blocking), so results
// agree with a real Eigen build to round-off, not bitwise.
#pragma once

#include <algorithm>
#include <cassert>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <limits>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
constexpr int Infinity = -1;
enum StorageOptions { ColMajor = 0, RowMajor = 1, AutoAlign = 0 };
enum DecompositionOptions { ComputeThinU = 1, ComputeFullU = 2, ComputeThinV = 4, ComputeFullV = 8 };

template <class S, int R, int C, int Opt = 0, int MR = R, int MC = C>
class Matrix;
template <class S, int R, int C>
class Block;

namespace internal {

template <class T>
struct traits {
  static constexpr bool dense = false;
};

// storage: inline for fixed sizes, heap for dynamic
template <int R, int C>
struct Storage {
  double d[(R > 0 ? R : 1) * (C > 0 ? C : 1)] = {};
  double* data() { return d; }
  const double* data() const { return d; }
  void resize(Index n) { assert(n == R * C); (void)n; }
  void swap(Storage& o) { std::swap(d, o.d); }
};
template <int R>
struct Storage<R, Dynamic> {
  std::vector<double> v;
  double* data() { return v.data(); }
  const double* data() const { return v.data(); }
  void resize(Index n) { v.assign(std::size_t(n), 0.0); }
  void swap(Storage& o) { v.swap(o.v); }
};
template <int C>
struct Storage<Dynamic, C> {
  std::vector<double> v;
  double* data() { return v.data(); }
  const double* data() const { return v.data(); }
  void resize(Index n) { v.assign(std::size_t(n), 0.0); }
  void swap(Storage& o) { v.swap(o.v); }
};
template <>
struct Storage<Dynamic, Dynamic> {
  std::vector<double> v;
  double* data() { return v.data(); }
  const double* data() const { return v.data(); }
  void resize(Index n) { v.assign(std::size_t(n), 0.0); }
  void swap(Storage& o) { v.swap(o.v); }
};

constexpr int pick(int a, int b) { return a != Dynamic ? a : b; }

}  // namespace internal

template <class T>
constexpr bool is_dense_v = internal::traits<std::decay_t<T>>::dense;

template <class Derived>
class ArrayWrapper;

/// Common interface of Matrix and Block: column-major strided memory.
template <class Derived>
class DenseBase {
 public:
  Derived& self() { return static_cast<Derived&>(*this); }
  const Derived& self() const { return static_cast<const Derived&>(*this); }

  Index size() const { return self().rows() * self().cols(); }
  double& operator()(Index i, Index j) { return self().data()[i + j * self().outerStride()]; }
  double operator()(Index i, Index j) const { return self().data()[i + j * self().outerStride()]; }
  double coeff(Index i, Index j) const { return (*this)(i, j); }
  double& coeffRef(Index i, Index j) { return (*this)(i, j); }
  // linear (vector) access: along the only non-unit dimension
  double& operator()(Index i) { return self().data()[lin(i)]; }
  double operator()(Index i) const { return self().data()[lin(i)]; }
  double& operator[](Index i) { return self().data()[lin(i)]; }
  double operator[](Index i) const { return self().data()[lin(i)]; }
  double& coeffRef(Index i) { return self().data()[lin(i)]; }
  double coeff(Index i) const { return self().data()[lin(i)]; }
  double x() const { return (*this)(0); }
  double y() const { return (*this)(1); }
  double& x() { return (*this)(0); }
  double& y() { return (*this)(1); }

  Index lin(Index i) const {
    if (self().cols() == 1) return i;
    if (self().rows() == 1) return i * self().outerStride();
    return (i % self().rows()) + (i / self().rows()) * self().outerStride();
  }

  // ---- views
  Block<double, Dynamic, Dynamic> block(Index i, Index j, Index r, Index c);
  Block<double, Dynamic, Dynamic> block(Index i, Index j, Index r, Index c) const;
  Block<double, Dynamic, 1> col(Index j);
  Block<double, Dynamic, 1> col(Index j) const;
  Block<double, 1, Dynamic> row(Index i);
  Block<double, 1, Dynamic> row(Index i) const;
  auto topRows(Index n) { return block(0, 0, n, self().cols()); }
  auto topRows(Index n) const { return block(0, 0, n, self().cols()); }
  auto bottomRows(Index n) { return block(self().rows() - n, 0, n, self().cols()); }
  auto bottomRows(Index n) const { return block(self().rows() - n, 0, n, self().cols()); }
  auto middleRows(Index s, Index n) { return block(s, 0, n, self().cols()); }
  auto middleRows(Index s, Index n) const { return block(s, 0, n, self().cols()); }
  auto leftCols(Index n) { return block(0, 0, self().rows(), n); }
  auto leftCols(Index n) const { return block(0, 0, self().rows(), n); }
  auto rightCols(Index n) { return block(0, self().cols() - n, self().rows(), n); }
  auto rightCols(Index n) const { return block(0, self().cols() - n, self().rows(), n); }
  auto middleCols(Index s, Index n) { return block(0, s, self().rows(), n); }
  auto middleCols(Index s, Index n) const { return block(0, s, self().rows(), n); }
  auto topLeftCorner(Index r, Index c) { return block(0, 0, r, c); }
  auto topLeftCorner(Index r, Index c) const { return block(0, 0, r, c); }
  auto topRightCorner(Index r, Index c) { return block(0, self().cols() - c, r, c); }
  auto topRightCorner(Index r, Index c) const { return block(0, self().cols() - c, r, c); }
  auto bottomLeftCorner(Index r, Index c) { return block(self().rows() - r, 0, r, c); }
  auto bottomLeftCorner(Index r, Index c) const { return block(self().rows() - r, 0, r, c); }
  auto bottomRightCorner(Index r, Index c) {
    return block(self().rows() - r, self().cols() - c, r, c);
  }
  auto bottomRightCorner(Index r, Index c) const {
    return block(self().rows() - r, self().cols() - c, r, c);
  }
  // vector segments keep the vector's orientation
  auto segment(Index s, Index n) {
    return self().cols() == 1 ? block(s, 0, n, 1) : block(0, s, 1, n);
  }
  auto segment(Index s, Index n) const {
    return self().cols() == 1 ? block(s, 0, n, 1) : block(0, s, 1, n);
  }
  auto head(Index n) { return segment(0, n); }
  auto head(Index n) const { return segment(0, n); }
  auto tail(Index n) { return segment(size() - n, n); }
  auto tail(Index n) const { return segment(size() - n, n); }

  // ---- reductions
  double sum() const {
    double s = 0;
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) s += (*this)(i, j);
    return s;
  }
  double squaredNorm() const {
    double s = 0;
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) s += (*this)(i, j) * (*this)(i, j);
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  template <int p>
  double lpNorm() const {
    static_assert(p == Infinity || p == 1 || p == 2, "lpNorm<p>");
    if (p == 2) return norm();
    double s = 0;
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i)
        s = p == Infinity ? std::max(s, std::abs((*this)(i, j))) : s + std::abs((*this)(i, j));
    return s;
  }
  template <class O>
  double dot(const DenseBase<O>& o) const {
    assert(size() == o.size());
    double s = 0;
    for (Index i = 0; i < size(); ++i) s += (*this)[i] * o[i];
    return s;
  }
  double maxCoeff() const {
    double m = -std::numeric_limits<double>::infinity();
    for (Index i = 0; i < size(); ++i) m = std::max(m, (*this)[i]);
    return m;
  }
  double minCoeff() const {
    double m = std::numeric_limits<double>::infinity();
    for (Index i = 0; i < size(); ++i) m = std::min(m, (*this)[i]);
    return m;
  }
  double trace() const {
    double s = 0;
    for (Index i = 0; i < std::min(self().rows(), self().cols()); ++i) s += (*this)(i, i);
    return s;
  }
  bool isZero(double prec = 1e-12) const {
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i)
        if (std::abs((*this)(i, j)) > prec) return false;
    return true;
  }
  bool allFinite() const {
    for (Index i = 0; i < size(); ++i)
      if (!std::isfinite((*this)[i])) return false;
    return true;
  }

  // ---- evaluated transforms (defined after Matrix)
  auto eval() const;
  auto transpose() const;
  auto normalized() const;
  auto cwiseAbs() const;
  template <class O>
  auto cwiseQuotient(const DenseBase<O>& o) const;
  template <class O>
  auto cwiseProduct(const DenseBase<O>& o) const;
  auto asDiagonal() const;
  double determinant() const;
  auto inverse() const;
  ArrayWrapper<Derived> array() { return ArrayWrapper<Derived>(self()); }
  auto lu() const;
  auto ldlt() const;
  auto fullPivLu() const;
  auto partialPivLu() const;

  // ---- in-place arithmetic
  void normalize() { self() /= norm(); }
  Derived& setZero() { return setConstant(0.0); }
  Derived& setOnes() { return setConstant(1.0); }
  Derived& setConstant(double v) {
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) (*this)(i, j) = v;
    return self();
  }
  Derived& setIdentity() {
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) (*this)(i, j) = i == j ? 1.0 : 0.0;
    return self();
  }
  Derived& fill(double v) { return setConstant(v); }
  Derived& operator*=(double a) {
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) (*this)(i, j) *= a;
    return self();
  }
  Derived& operator/=(double a) {
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) (*this)(i, j) /= a;
    return self();
  }
  template <class O>
  Derived& operator+=(const DenseBase<O>& o) {
    check(o);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) (*this)(i, j) += o(i, j);
    return self();
  }
  template <class O>
  Derived& operator-=(const DenseBase<O>& o) {
    check(o);
    for (Index j = 0; j < self().cols(); ++j)
      for (Index i = 0; i < self().rows(); ++i) (*this)(i, j) -= o(i, j);
    return self();
  }
  template <class O>
  void check(const DenseBase<O>& o) const {
    if (o.self().rows() != self().rows() || o.self().cols() != self().cols()) {
      // vectors of either orientation combine by linear index
      if (!(o.size() == size() && (self().rows() == 1 || self().cols() == 1)))
        throw std::logic_error("eigen shim: size mismatch");
    }
  }
};

template <class S, int R, int C>
class Block : public DenseBase<Block<S, R, C>> {
 public:
  using Base = DenseBase<Block<S, R, C>>;
  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;
  Block(double* p, Index r, Index c, Index os) : p_(p), r_(r), c_(c), os_(os) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index outerStride() const { return os_; }
  double* data() const { return p_; }

  Block& operator=(const Block& o) { return assign(o); }
  template <class O>
  Block& operator=(const DenseBase<O>& o) { return assign(o); }
  using Base::operator();
  using Base::operator[];

 private:
  template <class O>
  Block& assign(const DenseBase<O>& o) {
    // evaluate first: the source may alias this view
    std::vector<double> tmp(std::size_t(o.size()));
    if (o.self().rows() == r_ && o.self().cols() == c_) {
      for (Index j = 0; j < c_; ++j)
        for (Index i = 0; i < r_; ++i) tmp[std::size_t(i + j * r_)] = o(i, j);
      for (Index j = 0; j < c_; ++j)
        for (Index i = 0; i < r_; ++i) (*this)(i, j) = tmp[std::size_t(i + j * r_)];
    } else {
      this->check(o);
      for (Index i = 0; i < o.size(); ++i) tmp[std::size_t(i)] = o[i];
      for (Index i = 0; i < o.size(); ++i) (*this)[i] = tmp[std::size_t(i)];
    }
    return *this;
  }
  double* p_;
  Index r_, c_, os_;
};

template <class S, int R, int C>
struct internal::traits<Block<S, R, C>> {
  static constexpr bool dense = true;
  static constexpr int rows = R, cols = C;
};

template <class S, int R, int C, int Opt, int MR, int MC>
struct internal::traits<Matrix<S, R, C, Opt, MR, MC>> {
  static constexpr bool dense = true;
  static constexpr int rows = R, cols = C;
};

template <class S, int R, int C, int Opt, int MR, int MC>
class Matrix : public DenseBase<Matrix<S, R, C, Opt, MR, MC>> {
  static_assert(std::is_same<S, double>::value, "eigen shim: double only");

 public:
  using Base = DenseBase<Matrix>;
  using Scalar = double;
  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;
  static constexpr bool IsVector = (C == 1 || R == 1);

  Matrix() { init(R > 0 ? R : 0, C > 0 ? C : 0); }
  // Vec(n) / RowVec(n): size; only dynamic vectors
  template <class I, std::enable_if_t<std::is_integral<I>::value && IsVector && (R == Dynamic || C == Dynamic), int> = 0>
  explicit Matrix(I n) {
    init(C == 1 ? Index(n) : 1, C == 1 ? 1 : Index(n));
  }
  // dynamic matrix (rows, cols)
  template <class I, class J,
            std::enable_if_t<std::is_integral<I>::value && std::is_integral<J>::value &&
                                 !(R == 2 && C == 1),
                             int> = 0>
  Matrix(I r, J c) {
    init(R > 0 ? R : Index(r), C > 0 ? C : Index(c));
    if (R > 0 && C > 0 && (r != R || c != C)) throw std::logic_error("eigen shim: fixed size");
  }
  // fixed 2-vector coefficients
  template <class A, class B,
            std::enable_if_t<std::is_arithmetic<A>::value && std::is_arithmetic<B>::value && (R == 2 && C == 1),
                             int> = 0>
  Matrix(A a, B b) {
    init(2, 1);
    d_.data()[0] = double(a);
    d_.data()[1] = double(b);
  }
  // dense copy of a sparse matrix (Mat(sparse))
  template <class Sp, class = decltype(std::declval<const Sp&>().nonZeros()),
            std::enable_if_t<!is_dense_v<Sp>, int> = 0>
  explicit Matrix(const Sp& sp) {
    init(sp.rows(), sp.cols());
    for (Index o = 0; o < sp.outerSize(); ++o)
      for (typename Sp::InnerIterator it(sp, o); it; ++it) (*this)(it.row(), it.col()) += it.value();
  }
  Matrix(const Matrix& o) { copy_from(o); }
  Matrix(Matrix&& o) noexcept : r_(o.r_), c_(o.c_) { d_.swap(o.d_); }
  template <class O>
  Matrix(const DenseBase<O>& o) { copy_from(o); }
  Matrix& operator=(const Matrix& o) {
    if (this != &o) copy_from(o);
    return *this;
  }
  Matrix& operator=(Matrix&& o) noexcept {
    r_ = o.r_;
    c_ = o.c_;
    d_.swap(o.d_);
    return *this;
  }
  template <class O>
  Matrix& operator=(const DenseBase<O>& o) {
    Matrix tmp(o);
    *this = std::move(tmp);
    return *this;
  }

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index outerStride() const { return r_; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  using Base::operator();
  using Base::operator[];

  void resize(Index n) {
    if (C == 1) resize(n, 1);
    else resize(1, n);
  }
  void resize(Index r, Index c) {
    if (r == r_ && c == c_) return;
    init(r, c);
  }
  void swap(Matrix& o) {
    std::swap(r_, o.r_);
    std::swap(c_, o.c_);
    d_.swap(o.d_);
  }

  static Matrix Zero() { return Matrix(); }
  static Matrix Zero(Index n) { return Matrix(n).setZeroRet(); }
  static Matrix Zero(Index r, Index c) { return Matrix(r, c).setZeroRet(); }
  static Matrix Ones() { return Constant(1.0); }
  static Matrix Ones(Index n) { return Constant(n, 1.0); }
  static Matrix Ones(Index r, Index c) { return Constant(r, c, 1.0); }
  static Matrix Constant(double v) {
    Matrix m;
    m.setConstant(v);
    return m;
  }
  static Matrix Constant(Index n, double v) {
    Matrix m(n);
    m.setConstant(v);
    return m;
  }
  static Matrix Constant(Index r, Index c, double v) {
    Matrix m(r, c);
    m.setConstant(v);
    return m;
  }
  static Matrix Identity() {
    Matrix m;
    m.setIdentity();
    return m;
  }
  static Matrix Identity(Index r, Index c) {
    Matrix m(r, c);
    m.setIdentity();
    return m;
  }
  static Matrix Unit(Index n, Index i) {
    Matrix m = Zero(n);
    m[i] = 1.0;
    return m;
  }
  static Matrix UnitX() { return Unit(R, 0); }
  static Matrix UnitY() { return Unit(R, 1); }

  // comma initializer (row-major fill order, as Eigen)
  struct Comma {
    Matrix& m;
    Index k;
    Comma& operator,(double v) {
      m(k / m.cols(), k % m.cols()) = v;
      ++k;
      return *this;
    }
  };
  Comma operator<<(double v) {
    (*this)(0, 0) = v;
    return Comma{*this, 1};
  }

 private:
  Matrix setZeroRet() {
    this->setZero();
    return std::move(*this);
  }
  void init(Index r, Index c) {
    r_ = r;
    c_ = c;
    d_.resize(r * c);
  }
  template <class O>
  void copy_from(const DenseBase<O>& o) {
    Index r = o.self().rows(), c = o.self().cols();
    if (IsVector && (r == 1 || c == 1)) {  // vectors adopt this orientation
      Index n = r * c;
      if (C == 1) r = n, c = 1;
      else if (R == 1) r = 1, c = n;
    }
    std::vector<double> tmp(std::size_t(r * c));
    if (r == o.self().rows())
      for (Index j = 0; j < c; ++j)
        for (Index i = 0; i < r; ++i) tmp[std::size_t(i + j * r)] = o(i, j);
    else
      for (Index i = 0; i < r * c; ++i) tmp[std::size_t(i)] = o[i];
    init(r, c);
    std::copy(tmp.begin(), tmp.end(), d_.data());
  }
  internal::Storage<R, C> d_;
  Index r_ = 0, c_ = 0;
};

using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using RowVectorXd = Matrix<double, 1, Dynamic>;
using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Matrix2d = Matrix<double, 2, 2>;
using Matrix3d = Matrix<double, 3, 3>;

// ---- view constructors
template <class D>
Block<double, Dynamic, Dynamic> DenseBase<D>::block(Index i, Index j, Index r, Index c) {
  return {self().data() + i + j * self().outerStride(), r, c, self().outerStride()};
}
template <class D>
Block<double, Dynamic, Dynamic> DenseBase<D>::block(Index i, Index j, Index r, Index c) const {
  return {const_cast<double*>(self().data()) + i + j * self().outerStride(), r, c,
          self().outerStride()};
}
template <class D>
Block<double, Dynamic, 1> DenseBase<D>::col(Index j) {
  return {self().data() + j * self().outerStride(), self().rows(), 1, self().outerStride()};
}
template <class D>
Block<double, Dynamic, 1> DenseBase<D>::col(Index j) const {
  return {const_cast<double*>(self().data()) + j * self().outerStride(), self().rows(), 1,
          self().outerStride()};
}
template <class D>
Block<double, 1, Dynamic> DenseBase<D>::row(Index i) {
  return {self().data() + i, 1, self().cols(), self().outerStride()};
}
template <class D>
Block<double, 1, Dynamic> DenseBase<D>::row(Index i) const {
  return {const_cast<double*>(self().data()) + i, 1, self().cols(), self().outerStride()};
}

// ---- result types
namespace internal {
template <class A>
using plain_t = Matrix<double, traits<std::decay_t<A>>::rows, traits<std::decay_t<A>>::cols>;
template <class A, class B>
using sum_t = Matrix<double, pick(traits<std::decay_t<A>>::rows, traits<std::decay_t<B>>::rows),
                     pick(traits<std::decay_t<A>>::cols, traits<std::decay_t<B>>::cols)>;
template <class A, class B>
using prod_t = Matrix<double, traits<std::decay_t<A>>::rows, traits<std::decay_t<B>>::cols>;
template <class A>
using tr_t = Matrix<double, traits<std::decay_t<A>>::cols, traits<std::decay_t<A>>::rows>;
}  // namespace internal

template <class D>
auto DenseBase<D>::eval() const {
  return internal::plain_t<D>(*this);
}
template <class D>
auto DenseBase<D>::transpose() const {
  internal::tr_t<D> t(self().cols(), self().rows());
  for (Index j = 0; j < self().cols(); ++j)
    for (Index i = 0; i < self().rows(); ++i) t(j, i) = (*this)(i, j);
  return t;
}
template <class D>
auto DenseBase<D>::normalized() const {
  internal::plain_t<D> t(*this);
  t /= norm();
  return t;
}
template <class D>
auto DenseBase<D>::cwiseAbs() const {
  internal::plain_t<D> t(*this);
  for (Index i = 0; i < t.size(); ++i) t[i] = std::abs(t[i]);
  return t;
}
template <class D>
template <class O>
auto DenseBase<D>::cwiseQuotient(const DenseBase<O>& o) const {
  internal::plain_t<D> t(*this);
  for (Index i = 0; i < t.size(); ++i) t[i] /= o[i];
  return t;
}
template <class D>
template <class O>
auto DenseBase<D>::cwiseProduct(const DenseBase<O>& o) const {
  internal::plain_t<D> t(*this);
  for (Index i = 0; i < t.size(); ++i) t[i] *= o[i];
  return t;
}
template <class D>
auto DenseBase<D>::asDiagonal() const {
  MatrixXd m = MatrixXd::Zero(size(), size());
  for (Index i = 0; i < size(); ++i) m(i, i) = (*this)[i];
  return m;
}
template <class D>
double DenseBase<D>::determinant() const {
  const Index n = self().rows();
  if (n == 1) return (*this)(0, 0);
  if (n == 2) return (*this)(0, 0) * (*this)(1, 1) - (*this)(0, 1) * (*this)(1, 0);
  if (n == 3)
    return (*this)(0, 0) * ((*this)(1, 1) * (*this)(2, 2) - (*this)(1, 2) * (*this)(2, 1)) -
           (*this)(0, 1) * ((*this)(1, 0) * (*this)(2, 2) - (*this)(1, 2) * (*this)(2, 0)) +
           (*this)(0, 2) * ((*this)(1, 0) * (*this)(2, 1) - (*this)(1, 1) * (*this)(2, 0));
  throw std::logic_error("eigen shim: determinant for n <= 3 only");
}
template <class D>
auto DenseBase<D>::inverse() const {
  internal::plain_t<D> m(*this);
  const Index n = self().rows();
  if (n == 2) {
    const double det = determinant();
    m(0, 0) = (*this)(1, 1) / det;
    m(1, 1) = (*this)(0, 0) / det;
    m(0, 1) = -(*this)(0, 1) / det;
    m(1, 0) = -(*this)(1, 0) / det;
    return m;
  }
  throw std::logic_error("eigen shim: inverse for 2x2 only");
}

// ---- arithmetic operators
template <class A, class B, std::enable_if_t<is_dense_v<A> && is_dense_v<B>, int> = 0>
auto operator+(const A& a, const B& b) {
  internal::sum_t<A, B> t(a);
  t += b;
  return t;
}
template <class A, class B, std::enable_if_t<is_dense_v<A> && is_dense_v<B>, int> = 0>
auto operator-(const A& a, const B& b) {
  internal::sum_t<A, B> t(a);
  t -= b;
  return t;
}
template <class A, std::enable_if_t<is_dense_v<A>, int> = 0>
auto operator-(const A& a) {
  internal::plain_t<A> t(a);
  t *= -1.0;
  return t;
}
template <class A, class S,
          std::enable_if_t<is_dense_v<A> && std::is_arithmetic<S>::value, int> = 0>
auto operator*(const A& a, S s) {
  internal::plain_t<A> t(a);
  t *= double(s);
  return t;
}
template <class A, class S,
          std::enable_if_t<is_dense_v<A> && std::is_arithmetic<S>::value, int> = 0>
auto operator*(S s, const A& a) {
  internal::plain_t<A> t(a);
  for (Index i = 0; i < t.size(); ++i) t[i] = double(s) * t[i];
  return t;
}
template <class A, class S,
          std::enable_if_t<is_dense_v<A> && std::is_arithmetic<S>::value, int> = 0>
auto operator/(const A& a, S s) {
  internal::plain_t<A> t(a);
  t /= double(s);
  return t;
}
// matrix product (inner-product order per entry)
template <class A, class B, std::enable_if_t<is_dense_v<A> && is_dense_v<B>, int> = 0>
auto operator*(const A& a, const B& b) {
  if (a.cols() != b.rows()) throw std::logic_error("eigen shim: product size mismatch");
  internal::prod_t<A, B> t(a.rows(), b.cols());
  for (Index j = 0; j < b.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) {
      double s = 0;
      for (Index k = 0; k < a.cols(); ++k) s += a(i, k) * b(k, j);
      t(i, j) = s;
    }
  return t;
}

template <class A, std::enable_if_t<is_dense_v<A>, int> = 0>
bool operator==(const A& a, const A& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
  for (Index i = 0; i < a.size(); ++i)
    if (a[i] != b[i]) return false;
  return true;
}

template <class Derived>
class ArrayWrapper {
 public:
  explicit ArrayWrapper(Derived& d) : d_(d) {}
  ArrayWrapper& operator-=(double v) {
    for (Index i = 0; i < d_.size(); ++i) d_[i] -= v;
    return *this;
  }
  ArrayWrapper& operator+=(double v) {
    for (Index i = 0; i < d_.size(); ++i) d_[i] += v;
    return *this;
  }
  ArrayWrapper& operator*=(double v) {
    for (Index i = 0; i < d_.size(); ++i) d_[i] *= v;
    return *this;
  }
  Derived& matrix() { return d_; }

 private:
  Derived& d_;
};

// ------------------------------------------------------------------------
// Decompositions
// ------------------------------------------------------------------------

/// LU with partial (row) pivoting, P A = L U: column k pivots on the first
/// largest |a(i,k)|, i >= k (Eigen's unblocked PartialPivLU kernel).
template <class M>
class PartialPivLU {
 public:
  PartialPivLU() = default;
  template <class O>
  explicit PartialPivLU(const DenseBase<O>& a) {
    compute(a);
  }
  template <class O>
  PartialPivLU& compute(const DenseBase<O>& a) {
    lu_ = MatrixXd(a);
    const Index n = lu_.rows();
    perm_.resize(std::size_t(n));
    for (Index i = 0; i < n; ++i) perm_[std::size_t(i)] = i;
    for (Index k = 0; k < n; ++k) {
      Index p = k;
      double best = std::abs(lu_(k, k));
      for (Index i = k + 1; i < n; ++i)
        if (std::abs(lu_(i, k)) > best) best = std::abs(lu_(i, k)), p = i;
      if (p != k) {
        for (Index j = 0; j < n; ++j) std::swap(lu_(k, j), lu_(p, j));
        std::swap(perm_[std::size_t(k)], perm_[std::size_t(p)]);
      }
      const double piv = lu_(k, k);
      if (piv != 0.0)
        for (Index i = k + 1; i < n; ++i) lu_(i, k) /= piv;
      for (Index j = k + 1; j < n; ++j) {
        const double ukj = lu_(k, j);
        for (Index i = k + 1; i < n; ++i) lu_(i, j) -= lu_(i, k) * ukj;
      }
    }
    return *this;
  }
  template <class B>
  auto solve(const B& b) const {
    internal::plain_t<B> x(b);
    const Index n = lu_.rows();
    if (x.rows() != n) throw std::logic_error("eigen shim: LU solve size");
    std::vector<double> col(static_cast<std::size_t>(n));
    for (Index c = 0; c < x.cols(); ++c) {
      for (Index i = 0; i < n; ++i) col[std::size_t(i)] = b(perm_[std::size_t(i)], c);
      for (Index i = 0; i < n; ++i) {  // L (unit) forward
        double s = col[std::size_t(i)];
        for (Index k = 0; k < i; ++k) s -= lu_(i, k) * col[std::size_t(k)];
        col[std::size_t(i)] = s;
      }
      for (Index i = n - 1; i >= 0; --i) {  // U backward
        double s = col[std::size_t(i)];
        for (Index k = i + 1; k < n; ++k) s -= lu_(i, k) * col[std::size_t(k)];
        col[std::size_t(i)] = s / lu_(i, i);
      }
      for (Index i = 0; i < n; ++i) x(i, c) = col[std::size_t(i)];
    }
    return x;
  }
  /// Solver for A^T x = b: U^T L^T P x = b.
  struct Transposed {
    const PartialPivLU* lu;
    template <class B>
    auto solve(const B& b) const {
      internal::plain_t<B> x(b);
      const MatrixXd& F = lu->lu_;
      const Index n = F.rows();
      std::vector<double> col(static_cast<std::size_t>(n));
      for (Index c = 0; c < x.cols(); ++c) {
        for (Index i = 0; i < n; ++i) col[std::size_t(i)] = b(i, c);
        for (Index i = 0; i < n; ++i) {  // U^T forward
          double s = col[std::size_t(i)];
          for (Index k = 0; k < i; ++k) s -= F(k, i) * col[std::size_t(k)];
          col[std::size_t(i)] = s / F(i, i);
        }
        for (Index i = n - 1; i >= 0; --i) {  // L^T backward (unit)
          double s = col[std::size_t(i)];
          for (Index k = i + 1; k < n; ++k) s -= F(k, i) * col[std::size_t(k)];
          col[std::size_t(i)] = s;
        }
        for (Index i = 0; i < n; ++i) x(lu->perm_[std::size_t(i)], c) = col[std::size_t(i)];
      }
      return x;
    }
  };
  Transposed transpose() const { return Transposed{this}; }
  const MatrixXd& matrixLU() const { return lu_; }
  double determinant() const {
    double d = 1;
    for (Index i = 0; i < lu_.rows(); ++i) d *= lu_(i, i);
    std::vector<Index> p = perm_;
    for (std::size_t i = 0; i < p.size(); ++i)
      while (p[i] != Index(i)) {
        std::swap(p[i], p[std::size_t(p[i])]);
        d = -d;
      }
    return d;
  }
  Index rows() const { return lu_.rows(); }
  Index cols() const { return lu_.cols(); }

 private:
  MatrixXd lu_;
  std::vector<Index> perm_;  // row i of P A is row perm_[i] of A
};

/// LU with complete pivoting; rank decisions use Eigen's default threshold
/// (epsilon * min(rows, cols) relative to the largest pivot).
template <class M>
class FullPivLU {
 public:
  FullPivLU() = default;
  template <class O>
  explicit FullPivLU(const DenseBase<O>& a) {
    compute(a);
  }
  template <class O>
  FullPivLU& compute(const DenseBase<O>& a) {
    lu_ = MatrixXd(a);
    const Index m = lu_.rows(), n = lu_.cols(), d = std::min(m, n);
    rp_.resize(std::size_t(m));
    cp_.resize(std::size_t(n));
    for (Index i = 0; i < m; ++i) rp_[std::size_t(i)] = i;
    for (Index j = 0; j < n; ++j) cp_[std::size_t(j)] = j;
    maxpivot_ = 0;
    nonzero_ = 0;
    for (Index k = 0; k < d; ++k) {
      Index pr = k, pc = k;
      double best = -1;
      for (Index j = k; j < n; ++j)
        for (Index i = k; i < m; ++i)
          if (std::abs(lu_(i, j)) > best) best = std::abs(lu_(i, j)), pr = i, pc = j;
      if (best == 0.0) break;
      maxpivot_ = std::max(maxpivot_, best);
      ++nonzero_;
      if (pr != k) {
        for (Index j = 0; j < n; ++j) std::swap(lu_(k, j), lu_(pr, j));
        std::swap(rp_[std::size_t(k)], rp_[std::size_t(pr)]);
      }
      if (pc != k) {
        for (Index i = 0; i < m; ++i) std::swap(lu_(i, k), lu_(i, pc));
        std::swap(cp_[std::size_t(k)], cp_[std::size_t(pc)]);
      }
      for (Index i = k + 1; i < m; ++i) lu_(i, k) /= lu_(k, k);
      for (Index j = k + 1; j < n; ++j)
        for (Index i = k + 1; i < m; ++i) lu_(i, j) -= lu_(i, k) * lu_(k, j);
    }
    return *this;
  }
  double threshold() const {
    return std::numeric_limits<double>::epsilon() * double(std::min(lu_.rows(), lu_.cols()));
  }
  Index rank() const {
    Index r = 0;
    for (Index i = 0; i < nonzero_; ++i)
      if (std::abs(lu_(i, i)) > threshold() * maxpivot_) ++r;
    return r;
  }
  bool isInvertible() const { return lu_.rows() == lu_.cols() && rank() == lu_.rows(); }
  template <class B>
  auto solve(const B& b) const {
    const Index n = lu_.rows();
    internal::plain_t<B> x(lu_.cols(), b.cols());
    std::vector<double> col(static_cast<std::size_t>(n));
    for (Index c = 0; c < b.cols(); ++c) {
      for (Index i = 0; i < n; ++i) col[std::size_t(i)] = b(rp_[std::size_t(i)], c);
      for (Index i = 0; i < n; ++i)
        for (Index k = 0; k < i; ++k) col[std::size_t(i)] -= lu_(i, k) * col[std::size_t(k)];
      for (Index i = n - 1; i >= 0; --i) {
        double s = col[std::size_t(i)];
        for (Index k = i + 1; k < n; ++k) s -= lu_(i, k) * col[std::size_t(k)];
        col[std::size_t(i)] = s / lu_(i, i);
      }
      for (Index i = 0; i < n; ++i) x(cp_[std::size_t(i)], c) = col[std::size_t(i)];
    }
    return x;
  }

 private:
  MatrixXd lu_;
  std::vector<Index> rp_, cp_;
  double maxpivot_ = 0;
  Index nonzero_ = 0;
};

/// Symmetric LDL^T with diagonal pivoting (largest remaining |d|, as
/// Eigen's LDLT).
template <class M>
class LDLT {
 public:
  LDLT() = default;
  template <class O>
  explicit LDLT(const DenseBase<O>& a) {
    compute(a);
  }
  template <class O>
  LDLT& compute(const DenseBase<O>& a) {
    m_ = MatrixXd(a);
    const Index n = m_.rows();
    perm_.resize(std::size_t(n));
    for (Index i = 0; i < n; ++i) perm_[std::size_t(i)] = i;
    for (Index k = 0; k < n; ++k) {
      Index p = k;
      for (Index i = k + 1; i < n; ++i)
        if (std::abs(m_(i, i)) > std::abs(m_(p, p))) p = i;
      if (p != k) {  // symmetric swap of rows/cols k and p
        for (Index j = 0; j < n; ++j) std::swap(m_(k, j), m_(p, j));
        for (Index i = 0; i < n; ++i) std::swap(m_(i, k), m_(i, p));
        std::swap(perm_[std::size_t(k)], perm_[std::size_t(p)]);
      }
      const double dk = m_(k, k);
      for (Index i = k + 1; i < n; ++i) {
        const double lik = dk != 0.0 ? m_(i, k) / dk : 0.0;
        for (Index j = k + 1; j <= i; ++j) {
          m_(i, j) -= lik * m_(j, k);
          m_(j, i) = m_(i, j);
        }
      }
      for (Index i = k + 1; i < n; ++i) m_(i, k) = dk != 0.0 ? m_(i, k) / dk : 0.0;
    }
    return *this;
  }
  template <class B>
  auto solve(const B& b) const {
    internal::plain_t<B> x(b);
    const Index n = m_.rows();
    std::vector<double> col(static_cast<std::size_t>(n));
    for (Index c = 0; c < x.cols(); ++c) {
      for (Index i = 0; i < n; ++i) col[std::size_t(i)] = b(perm_[std::size_t(i)], c);
      for (Index i = 0; i < n; ++i)
        for (Index k = 0; k < i; ++k) col[std::size_t(i)] -= m_(i, k) * col[std::size_t(k)];
      for (Index i = 0; i < n; ++i) col[std::size_t(i)] = m_(i, i) != 0.0 ? col[std::size_t(i)] / m_(i, i) : 0.0;
      for (Index i = n - 1; i >= 0; --i)
        for (Index k = i + 1; k < n; ++k) col[std::size_t(i)] -= m_(k, i) * col[std::size_t(k)];
      for (Index i = 0; i < n; ++i) x(perm_[std::size_t(i)], c) = col[std::size_t(i)];
    }
    return x;
  }
  int info() const { return 0; }

 private:
  MatrixXd m_;
  std::vector<Index> perm_;
};

/// Singular value decomposition by one-sided (Hestenes) Jacobi rotations,
/// singular values sorted decreasingly; full U / V completed to orthonormal
/// bases. solve() is the minimum-norm least-squares solution over the
/// singular values above Eigen's default threshold (diag size * epsilon
/// relative to the largest).
template <class M>
class JacobiSVD {
 public:
  JacobiSVD() = default;
  template <class O>
  JacobiSVD(const DenseBase<O>& a, unsigned = 0) {
    compute(MatrixXd(a));
  }
  const VectorXd& singularValues() const { return s_; }
  const MatrixXd& matrixU() const { return U_; }
  const MatrixXd& matrixV() const { return V_; }
  Index rank() const {
    if (s_.size() == 0) return 0;
    const double thr = std::max(s_[0] * double(s_.size()) * std::numeric_limits<double>::epsilon(),
                                std::numeric_limits<double>::min());
    Index r = 0;
    for (Index i = 0; i < s_.size(); ++i)
      if (s_[i] > thr) ++r;
    return r;
  }
  template <class B>
  auto solve(const B& b) const {
    const Index r = rank();
    internal::plain_t<B> x(V_.rows(), b.cols());
    for (Index c = 0; c < b.cols(); ++c) {
      VectorXd t(r);
      for (Index i = 0; i < r; ++i) {
        double s = 0;
        for (Index k = 0; k < U_.rows(); ++k) s += U_(k, i) * b(k, c);
        t[i] = s / s_[i];
      }
      for (Index j = 0; j < V_.rows(); ++j) {
        double s = 0;
        for (Index i = 0; i < r; ++i) s += V_(j, i) * t[i];
        x(j, c) = s;
      }
    }
    return x;
  }

 private:
  // one-sided Jacobi on the columns of A (m >= n): A V = W, W_j = s_j u_j
  static void hestenes(MatrixXd& W, MatrixXd& V) {
    const Index n = W.cols(), m = W.rows();
    V = MatrixXd::Identity(n, n);
    for (int sweep = 0; sweep < 100; ++sweep) {
      bool rotated = false;
      for (Index p = 0; p < n; ++p)
        for (Index q = p + 1; q < n; ++q) {
          double a = 0, b = 0, g = 0;
          for (Index i = 0; i < m; ++i) {
            a += W(i, p) * W(i, p);
            b += W(i, q) * W(i, q);
            g += W(i, p) * W(i, q);
          }
          if (std::abs(g) <= 1e-15 * std::sqrt(a * b) || g == 0.0) continue;
          rotated = true;
          const double zeta = (b - a) / (2 * g);
          const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1 + zeta * zeta));
          const double c = 1 / std::sqrt(1 + t * t), s = c * t;
          for (Index i = 0; i < m; ++i) {
            const double wp = W(i, p), wq = W(i, q);
            W(i, p) = c * wp - s * wq;
            W(i, q) = s * wp + c * wq;
          }
          for (Index i = 0; i < n; ++i) {
            const double vp = V(i, p), vq = V(i, q);
            V(i, p) = c * vp - s * vq;
            V(i, q) = s * vp + c * vq;
          }
        }
      if (!rotated) break;
    }
  }
  // extends the first `have` orthonormal columns of Q (m x m) to a basis
  static void complete(MatrixXd& Q, Index have) {
    const Index m = Q.rows();
    Index col = have;
    for (Index e = 0; e < m && col < m; ++e) {
      VectorXd v = VectorXd::Zero(m);
      v[e] = 1.0;
      for (int pass = 0; pass < 2; ++pass)
        for (Index j = 0; j < col; ++j) {
          double d = 0;
          for (Index i = 0; i < m; ++i) d += Q(i, j) * v[i];
          for (Index i = 0; i < m; ++i) v[i] -= d * Q(i, j);
        }
      const double nv = v.norm();
      if (nv < 1e-8) continue;
      for (Index i = 0; i < m; ++i) Q(i, col) = v[i] / nv;
      ++col;
    }
  }
  void compute(const MatrixXd& A) {
    const bool tr = A.rows() < A.cols();
    MatrixXd W = tr ? MatrixXd(A.transpose()) : A;  // tall: m >= n
    MatrixXd Vs;
    hestenes(W, Vs);
    const Index m = W.rows(), n = W.cols();
    std::vector<Index> order(static_cast<std::size_t>(n));
    std::vector<double> sv(static_cast<std::size_t>(n));
    for (Index j = 0; j < n; ++j) {
      order[std::size_t(j)] = j;
      double s = 0;
      for (Index i = 0; i < m; ++i) s += W(i, j) * W(i, j);
      sv[std::size_t(j)] = std::sqrt(s);
    }
    std::stable_sort(order.begin(), order.end(),
                     [&](Index a, Index b) { return sv[std::size_t(a)] > sv[std::size_t(b)]; });
    s_ = VectorXd(n);
    MatrixXd Ut = MatrixXd::Zero(m, m), Vt(n, n);
    Index nz = 0;
    for (Index j = 0; j < n; ++j) {
      const Index o = order[std::size_t(j)];
      s_[j] = sv[std::size_t(o)];
      for (Index i = 0; i < n; ++i) Vt(i, j) = Vs(i, o);
      if (s_[j] > 1e-300 && s_[j] > 1e-14 * s_[0]) {
        for (Index i = 0; i < m; ++i) Ut(i, j) = W(i, o) / s_[j];
        nz = j + 1;
      }
    }
    complete(Ut, nz);  // left vectors of zero singular values + the rest
    if (!tr) {
      U_ = Ut;
      V_ = Vt;
    } else {  // A^T = Ut S Vt^T  =>  A = Vt S Ut^T
      U_ = Vt;
      V_ = Ut;
    }
  }
  VectorXd s_;
  MatrixXd U_, V_;
};

template <class D>
auto DenseBase<D>::lu() const {
  return PartialPivLU<MatrixXd>(*this);
}
template <class D>
auto DenseBase<D>::partialPivLu() const {
  return PartialPivLU<MatrixXd>(*this);
}
template <class D>
auto DenseBase<D>::fullPivLu() const {
  return FullPivLU<MatrixXd>(*this);
}
template <class D>
auto DenseBase<D>::ldlt() const {
  return LDLT<MatrixXd>(*this);
}

}  // namespace Eigen
