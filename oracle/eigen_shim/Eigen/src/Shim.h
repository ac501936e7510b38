// Shim.h — TEST INFRASTRUCTURE ONLY.  A minimal, dependency-free subset of the Eigen 3 dense
// API, just enough to compile the UNMODIFIED reference sources
// (/root/reference/proj/src/{gait,robot,mpc,csc,ruiz,qp,ldl,batch,env,policy,ppo}.cpp) into
// oracle/_ref/, which pins the repo's restated oracle (oracle/rmpc_oracle*.hpp) to numbers the
// reference code itself produces.  Eigen 3 (proj/CMakeLists.txt:11) is absent from this image
// and there is no network, so the reference cannot be built against the real library.
//
// Semantics follow Eigen where the reference relies on them:
//   * column-major storage, fixed-size types hold their coefficients inline;
//   * block expressions (row/col/block/segment/head/tail/topRows/leftCols/transpose) are
//     writable views into the parent's storage, so `J.col(a) = ...`, `q.row(i).setZero()` and
//     `const auto x = b.head(n)` behave as in Eigen;
//   * every arithmetic expression is evaluated eagerly into a Matrix of the statically known
//     result size (no expression templates; assignment therefore never aliases);
//   * the comma initializer fills in row-major order;
//   * array() exposes coefficient-wise arithmetic.
// Rounding can differ from Eigen's in the last bits (Eigen unrolls fixed-size reductions as
// pairwise trees and vectorises); the reference's numerics do not depend on that.
// AMDOrdering is NOT Eigen's AMD: it forwards to the oracle's approximate-minimum-degree
// ordering (oracle/rmpc_oracle.hpp, min_degree_ordering), see OrderingMethods.
#pragma once

#include <algorithm>
#include <array>
#include <cassert>
#include <cmath>
#include <cstddef>
#include <limits>
#include <memory>
#include <stdexcept>
#include <type_traits>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
enum StorageOptions { ColMajor = 0, RowMajor = 1, AutoAlign = 0, DontAlign = 2 };
enum { Infinity = -1 };

namespace internal {
constexpr int pick(int a, int b) { return a != Dynamic ? a : b; }
inline void check(bool ok, const char* what) {
  if (!ok) throw std::logic_error(what);
}
}  // namespace internal

template <class Derived>
struct DenseBase;
template <int R, int C>
struct View;
template <class S, int R, int C, int Opt = 0, int MR = R, int MC = C>
class Matrix;
template <int R, int C>
struct ArrayWrap;

template <int R, int C>
using Result = Matrix<double, R, C>;

// compile-time shape of every dense type (read by the CRTP base before the type is complete)
template <class D>
struct traits;
template <int R, int C>
struct traits<View<R, C>> {
  static constexpr int Rows = R, Cols = C;
};
template <class S, int R, int C, int O, int MR, int MC>
struct traits<Matrix<S, R, C, O, MR, MC>> {
  static constexpr int Rows = R, Cols = C;
};
struct SizeTag {};
// View<R, C> made dependent on a defaulted template parameter, so DenseBase<View<..>> can declare
// (and define in-class) members that return views of its own type
template <int K, int R, int C>
using DView = std::conditional_t<(K >= 0), View<R, C>, void>;

// ---------------------------------------------------------------- comma initializer
template <class D>
struct CommaInit {
  D& m;
  Index k;
  CommaInit& operator,(double v) {
    const Index c = m.cols();
    m.ref(k / c, k % c) = v;
    ++k;
    return *this;
  }
  template <class O>
  CommaInit& operator,(const DenseBase<O>& o) {  // block-wise (vectors only, in order)
    for (Index i = 0; i < o.size(); ++i) (*this), o.lin(i);
    return *this;
  }
  D& finished() { return m; }
  operator D&() { return m; }
};

// ---------------------------------------------------------------- dense base (CRTP)
// Every dense object owns or views strided storage: coefficient (i, j) lives at
// data()[i * rstride() + j * cstride()].
template <class Derived>
struct DenseBase {
  static constexpr int Rows = traits<Derived>::Rows;
  static constexpr int Cols = traits<Derived>::Cols;
  const Derived& derived() const { return static_cast<const Derived&>(*this); }
  Derived& derived() { return static_cast<Derived&>(*this); }

  Index rows() const { return derived().rows_(); }
  Index cols() const { return derived().cols_(); }
  Index size() const { return rows() * cols(); }
  double* dptr() const { return derived().dptr_(); }
  Index rs() const { return derived().rs_(); }
  Index cs() const { return derived().cs_(); }
  double& ref(Index i, Index j) const { return dptr()[i * rs() + j * cs()]; }
  double coeff(Index i, Index j) const { return ref(i, j); }
  // linear (vector) index
  double& lin(Index k) const { return rows() == 1 ? ref(0, k) : (cols() == 1 ? ref(k, 0) : ref(k % rows(), k / rows())); }

  double& operator()(Index i, Index j) { return ref(i, j); }
  const double& operator()(Index i, Index j) const { return ref(i, j); }
  double& operator()(Index k) { return lin(k); }
  const double& operator()(Index k) const { return lin(k); }
  double& operator[](Index k) { return lin(k); }
  const double& operator[](Index k) const { return lin(k); }
  double& x() { return lin(0); }
  double& y() { return lin(1); }
  double x() const { return lin(0); }
  double y() const { return lin(1); }

  // ---- views
  template <int K = 0>
  DView<K, 1, Cols> row(Index i) const { return DView<K, 1, Cols>(&ref(i, 0), 1, cols(), rs(), cs()); }
  template <int K = 0>
  DView<K, Rows, 1> col(Index j) const { return DView<K, Rows, 1>(&ref(0, j), rows(), 1, rs(), cs()); }
  template <int BR, int BC>
  View<BR, BC> block(Index i, Index j) const { return View<BR, BC>(&ref(i, j), BR, BC, rs(), cs()); }
  template <int K = 0>
  DView<K, Dynamic, Dynamic> block(Index i, Index j, Index br, Index bc) const {
    return DView<K, Dynamic, Dynamic>(br ? &ref(i, j) : dptr(), br, bc, rs(), cs());
  }
  static constexpr bool kRowVec = Rows == 1;
  template <int K>
  using SegDyn = DView<K, (Rows == 1 ? 1 : Dynamic), (Rows == 1 ? Dynamic : 1)>;
  template <int N>
  using SegFix = View<(Rows == 1 ? 1 : N), (Rows == 1 ? N : 1)>;
  template <int K = 0>
  SegDyn<K> segment(Index k, Index n) const {
    if (rows() == 1) return SegDyn<K>(n ? &ref(0, k) : dptr(), 1, n, rs(), cs());
    return SegDyn<K>(n ? &ref(k, 0) : dptr(), n, 1, rs(), cs());
  }
  template <int N>
  SegFix<N> segment(Index k) const {
    if (rows() == 1) return SegFix<N>(&ref(0, k), 1, N, rs(), cs());
    return SegFix<N>(&ref(k, 0), N, 1, rs(), cs());
  }
  template <int K = 0>
  SegDyn<K> head(Index n) const { return segment<K>(0, n); }
  template <int K = 0>
  SegDyn<K> tail(Index n) const { return segment<K>(size() - n, n); }
  template <int N>
  SegFix<N> head() const { return segment<N>(0); }
  template <int N>
  SegFix<N> tail() const { return segment<N>(size() - N); }
  template <int N>
  View<N, Cols> topRows() const { return View<N, Cols>(dptr(), N, cols(), rs(), cs()); }
  template <int K = 0>
  DView<K, Dynamic, Cols> topRows(Index n) const { return DView<K, Dynamic, Cols>(dptr(), n, cols(), rs(), cs()); }
  template <int N>
  View<N, Cols> bottomRows() const { return View<N, Cols>(&ref(rows() - N, 0), N, cols(), rs(), cs()); }
  template <int N>
  View<Rows, N> leftCols() const { return View<Rows, N>(dptr(), rows(), N, rs(), cs()); }
  template <int K = 0>
  DView<K, Rows, Dynamic> leftCols(Index n) const { return DView<K, Rows, Dynamic>(dptr(), rows(), n, rs(), cs()); }
  template <int N>
  View<Rows, N> rightCols() const { return View<Rows, N>(&ref(0, cols() - N), rows(), N, rs(), cs()); }
  template <int K = 0>
  DView<K, Cols, Rows> transpose() const { return DView<K, Cols, Rows>(dptr(), cols(), rows(), cs(), rs()); }

  // ---- reductions
  double sum() const {
    double s = 0.0;
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) s += coeff(i, j);
    return s;
  }
  double squaredNorm() const {
    double s = 0.0;
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) s += coeff(i, j) * coeff(i, j);
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  double maxCoeff() const {
    double m = -std::numeric_limits<double>::infinity();
    for (Index k = 0; k < size(); ++k) m = std::max(m, lin(k));
    return m;
  }
  double minCoeff() const {
    double m = std::numeric_limits<double>::infinity();
    for (Index k = 0; k < size(); ++k) m = std::min(m, lin(k));
    return m;
  }
  template <int P>
  double lpNorm() const {
    static_assert(P == Infinity || P == 1 || P == 2, "lpNorm: Infinity, 1 or 2");
    if constexpr (P == Infinity) {
      double m = 0.0;
      for (Index k = 0; k < size(); ++k) m = std::max(m, std::abs(lin(k)));
      return m;
    } else if constexpr (P == 1) {
      double s = 0.0;
      for (Index k = 0; k < size(); ++k) s += std::abs(lin(k));
      return s;
    } else {
      return norm();
    }
  }
  bool allFinite() const {
    for (Index k = 0; k < size(); ++k)
      if (!std::isfinite(lin(k))) return false;
    return true;
  }
  bool hasNaN() const {
    for (Index k = 0; k < size(); ++k)
      if (std::isnan(lin(k))) return true;
    return false;
  }
  template <class O>
  double dot(const DenseBase<O>& o) const {
    internal::check(size() == o.size(), "dot: size mismatch");
    double s = 0.0;
    for (Index k = 0; k < size(); ++k) s += lin(k) * o.lin(k);
    return s;
  }

  // ---- coefficient-wise
  template <class F>
  Result<Rows, Cols> unaryExpr(F f) const {
    Result<Rows, Cols> r(rows(), cols(), SizeTag{});
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) r.ref(i, j) = f(coeff(i, j));
    return r;
  }
  template <class O, class F>
  Result<internal::pick(Rows, O::Rows), internal::pick(Cols, O::Cols)> binaryExpr(const DenseBase<O>& o, F f) const {
    internal::check(rows() == o.rows() && cols() == o.cols(), "coefficient-wise op: size mismatch");
    Result<internal::pick(Rows, O::Rows), internal::pick(Cols, O::Cols)> r(rows(), cols(), SizeTag{});
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) r.ref(i, j) = f(coeff(i, j), o.coeff(i, j));
    return r;
  }
  template <class O>
  auto cwiseProduct(const DenseBase<O>& o) const { return binaryExpr(o, [](double a, double b) { return a * b; }); }
  template <class O>
  auto cwiseQuotient(const DenseBase<O>& o) const { return binaryExpr(o, [](double a, double b) { return a / b; }); }
  template <class O>
  auto cwiseMax(const DenseBase<O>& o) const {
    return binaryExpr(o, [](double a, double b) { return a < b ? b : a; });
  }
  template <class O>
  auto cwiseMin(const DenseBase<O>& o) const {
    return binaryExpr(o, [](double a, double b) { return b < a ? b : a; });
  }
  Result<Rows, Cols> cwiseMax(double v) const { return unaryExpr([v](double a) { return a < v ? v : a; }); }
  Result<Rows, Cols> cwiseMin(double v) const { return unaryExpr([v](double a) { return v < a ? v : a; }); }
  Result<Rows, Cols> cwiseAbs() const { return unaryExpr([](double a) { return std::abs(a); }); }
  Result<Rows, Cols> cwiseSqrt() const { return unaryExpr([](double a) { return std::sqrt(a); }); }
  Result<Rows, Cols> eval() const { return Result<Rows, Cols>(derived()); }
  ArrayWrap<Rows, Cols> array() const { return ArrayWrap<Rows, Cols>(dptr(), rows(), cols(), rs(), cs()); }

  // ---- writes through (views and matrices alike)
  void fill_with(double v) const {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) ref(i, j) = v;
  }
  template <class O>
  void assign_from(const DenseBase<O>& o) const {
    if (rows() != o.rows() && (rows() == 1 || cols() == 1) && (o.rows() == 1 || o.cols() == 1) &&
        size() == o.size()) {  // Eigen transposes vectors on assignment
      for (Index k = 0; k < size(); ++k) lin(k) = o.lin(k);
      return;
    }
    internal::check(rows() == o.rows() && cols() == o.cols(), "assignment: size mismatch");
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) ref(i, j) = o.coeff(i, j);
  }
  template <class O>
  void add_from(const DenseBase<O>& o, double s) const {
    internal::check(rows() == o.rows() && cols() == o.cols(), "compound assignment: size mismatch");
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) ref(i, j) += s * o.coeff(i, j);
  }
  void scale_by(double s) const {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) ref(i, j) *= s;
  }
  void div_by(double s) const {
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) ref(i, j) /= s;
  }
};

// ---------------------------------------------------------------- strided view
template <int R, int C>
struct View : DenseBase<View<R, C>> {
  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;
  double* d;
  Index r, c, rstr, cstr;
  View(double* d_, Index r_, Index c_, Index rs_, Index cs_) : d(d_), r(r_), c(c_), rstr(rs_), cstr(cs_) {}
  View(const View&) = default;
  Index rows_() const { return r; }
  Index cols_() const { return c; }
  double* dptr_() const { return d; }
  Index rs_() const { return rstr; }
  Index cs_() const { return cstr; }
  double* data() const { return d; }

  const View& operator=(const View& o) const {
    Result<R, C> tmp(o);
    this->assign_from(tmp);
    return *this;
  }
  template <class O>
  const View& operator=(const DenseBase<O>& o) const {
    Result<R, C> tmp(o.derived());
    this->assign_from(tmp);
    return *this;
  }
  template <class O>
  const View& operator+=(const DenseBase<O>& o) const {
    Result<R, C> tmp(o.derived());
    this->add_from(tmp, 1.0);
    return *this;
  }
  template <class O>
  const View& operator-=(const DenseBase<O>& o) const {
    Result<R, C> tmp(o.derived());
    this->add_from(tmp, -1.0);
    return *this;
  }
  const View& operator*=(double s) const { this->scale_by(s); return *this; }
  const View& operator/=(double s) const { this->div_by(s); return *this; }
  const View& setZero() const { this->fill_with(0.0); return *this; }
  const View& setOnes() const { this->fill_with(1.0); return *this; }
  const View& setConstant(double v) const { this->fill_with(v); return *this; }
  const View& noalias() const { return *this; }
};

// Eigen::Map<MatrixType>: a view of caller memory.
template <class MT>
struct Map : View<MT::RowsAtCompileTime, MT::ColsAtCompileTime> {
  using Base = View<MT::RowsAtCompileTime, MT::ColsAtCompileTime>;
  Map(double* p, Index n)
      : Base(p, MT::ColsAtCompileTime == 1 ? n : 1, MT::ColsAtCompileTime == 1 ? 1 : n, 1,
             MT::ColsAtCompileTime == 1 ? n : 1) {}
  Map(const double* p, Index n) : Map(const_cast<double*>(p), n) {}
  Map(double* p, Index r_, Index c_) : Base(p, r_, c_, 1, r_) {}
  Map(const double* p, Index r_, Index c_) : Map(const_cast<double*>(p), r_, c_) {}
  Map(double* p) : Base(p, MT::RowsAtCompileTime, MT::ColsAtCompileTime, 1, MT::RowsAtCompileTime) {}
  Map(const double* p) : Map(const_cast<double*>(p)) {}
  using Base::operator=;
};

// ---------------------------------------------------------------- matrix
template <class S, int R, int C, int Opt, int MR, int MC>
class Matrix : public DenseBase<Matrix<S, R, C, Opt, MR, MC>> {
  static_assert(std::is_same_v<S, double>, "Eigen shim: double scalars only");
  static constexpr bool kFixed = R > 0 && C > 0;
  using Store = std::conditional_t<kFixed, std::array<double, (kFixed ? R * C : 1)>, std::vector<double>>;
  Store v_{};
  Index r_ = R > 0 ? R : 0, c_ = C > 0 ? C : 0;

 public:
  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;
  static constexpr int SizeAtCompileTime = kFixed ? R * C : Dynamic;
  using Scalar = double;
  Index rows_() const { return r_; }
  Index cols_() const { return c_; }
  double* dptr_() const { return const_cast<double*>(v_.data()); }
  Index rs_() const { return 1; }
  Index cs_() const { return r_; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }

  Matrix() {
    if constexpr (kFixed) v_.fill(0.0);
  }
  Matrix(const Matrix&) = default;
  Matrix(Matrix&&) = default;
  Matrix& operator=(const Matrix&) = default;
  Matrix& operator=(Matrix&&) = default;
  // sized, zero-filled (internal) constructor
  Matrix(Index r, Index c, SizeTag) { resize(r, c); }
  // Eigen: Vec(n) sizes a dynamic vector; VecN(x) for N == 1 would set a coefficient
  explicit Matrix(Index n) {
    if constexpr (kFixed) {
      static_assert(!kFixed || R * C == 1, "fixed-size single-argument constructor");
      v_[0] = (double)n;
    } else {
      if (C == 1 || (R != 1 && C == Dynamic && R == Dynamic)) resize(n, 1); else resize(1, n);
    }
  }
  // two arguments: coefficients of a fixed 2-vector, or (rows, cols) of a dynamic matrix
  template <class A, class B, std::enable_if_t<std::is_arithmetic_v<A> && std::is_arithmetic_v<B>, int> = 0>
  Matrix(A a, B b) {
    if constexpr (kFixed) {
      static_assert(!kFixed || R * C == 2, "fixed-size two-argument constructor");
      v_[0] = (double)a;
      v_[1] = (double)b;
    } else {
      resize((Index)a, (Index)b);
    }
  }
  Matrix(double a, double b, double c) {
    static_assert(kFixed && R * C == 3, "three-argument constructor");
    v_[0] = a; v_[1] = b; v_[2] = c;
  }
  Matrix(double a, double b, double c, double d) {
    static_assert(kFixed && R * C == 4, "four-argument constructor");
    v_[0] = a; v_[1] = b; v_[2] = c; v_[3] = d;
  }
  template <class O>
  Matrix(const DenseBase<O>& o) {
    const bool vt = (R == 1 && o.cols() == 1 && o.rows() != 1) || (C == 1 && o.rows() == 1 && o.cols() != 1);
    if (vt) {  // Eigen transposes vectors on assignment
      resize(R == 1 ? 1 : o.size(), R == 1 ? o.size() : 1);
      for (Index k = 0; k < o.size(); ++k) this->lin(k) = o.lin(k);
      return;
    }
    resize(o.rows(), o.cols());
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) this->ref(i, j) = o.coeff(i, j);
  }
  template <class O>
  Matrix& operator=(const DenseBase<O>& o) {
    Matrix tmp(o);  // evaluate first: the source may view this matrix
    *this = std::move(tmp);
    return *this;
  }

  void resize(Index r, Index c) {
    if constexpr (kFixed) {
      internal::check(r == R && c == C, "resize of a fixed-size matrix");
    } else {
      internal::check((R == Dynamic || r == R) && (C == Dynamic || c == C), "resize: fixed dimension");
      r_ = r;
      c_ = c;
      v_.assign((size_t)(r * c), 0.0);
    }
  }
  void resize(Index n) {
    if constexpr (C == 1) resize(n, 1);
    else if constexpr (R == 1) resize(1, n);
    else resize(n, 1);
  }
  void conservativeResize(Index n) {
    Matrix old = *this;
    resize(n);
    for (Index k = 0; k < std::min(n, old.size()); ++k) this->lin(k) = old.lin(k);
  }
  Matrix& setZero() { this->fill_with(0.0); return *this; }
  Matrix& setZero(Index n) { resize(n); return *this; }
  Matrix& setZero(Index r, Index c) { resize(r, c); return *this; }
  Matrix& setOnes() { this->fill_with(1.0); return *this; }
  Matrix& setOnes(Index n) { resize(n); this->fill_with(1.0); return *this; }
  Matrix& setConstant(double v) { this->fill_with(v); return *this; }
  Matrix& setConstant(Index n, double v) { resize(n); this->fill_with(v); return *this; }
  Matrix& setIdentity() {
    this->fill_with(0.0);
    for (Index k = 0; k < std::min(r_, c_); ++k) this->ref(k, k) = 1.0;
    return *this;
  }
  Matrix& noalias() { return *this; }

  static Matrix Zero() { return Matrix(R, C, SizeTag{}); }
  static Matrix Zero(Index n) { Matrix m; m.resize(n); return m; }
  static Matrix Zero(Index r, Index c) { return Matrix(r, c, SizeTag{}); }
  static Matrix Ones() { Matrix m(R, C, SizeTag{}); m.fill_with(1.0); return m; }
  static Matrix Ones(Index n) { Matrix m = Zero(n); m.fill_with(1.0); return m; }
  static Matrix Ones(Index r, Index c) { Matrix m(r, c, SizeTag{}); m.fill_with(1.0); return m; }
  static Matrix Constant(double v) { Matrix m(R, C, SizeTag{}); m.fill_with(v); return m; }
  static Matrix Constant(Index n, double v) { Matrix m = Zero(n); m.fill_with(v); return m; }
  static Matrix Constant(Index r, Index c, double v) { Matrix m(r, c, SizeTag{}); m.fill_with(v); return m; }
  static Matrix Identity() { Matrix m(R, C, SizeTag{}); m.setIdentity(); return m; }
  static Matrix Identity(Index r, Index c) { Matrix m(r, c, SizeTag{}); m.setIdentity(); return m; }

  template <class O>
  Matrix& operator+=(const DenseBase<O>& o) {
    Matrix tmp(o);
    this->add_from(tmp, 1.0);
    return *this;
  }
  template <class O>
  Matrix& operator-=(const DenseBase<O>& o) {
    Matrix tmp(o);
    this->add_from(tmp, -1.0);
    return *this;
  }
  Matrix& operator*=(double s) { this->scale_by(s); return *this; }
  Matrix& operator/=(double s) { this->div_by(s); return *this; }

  CommaInit<Matrix> operator<<(double v) {
    CommaInit<Matrix> ci{*this, 0};
    ci, v;
    return ci;
  }

  class LLTResult;
  LLTResult llt() const { return LLTResult(*this); }
};

// Cholesky A = L L^T of an SPD matrix (Eigen::LLT, lower), solve by two triangular sweeps.
template <class S, int R, int C, int Opt, int MR, int MC>
class Matrix<S, R, C, Opt, MR, MC>::LLTResult {
  Matrix<double, R, C> L_;
  bool ok_ = true;

 public:
  explicit LLTResult(const Matrix& a) : L_(a) {
    const Index n = a.rows();
    for (Index j = 0; j < n; ++j) {
      double d = L_(j, j);
      for (Index k = 0; k < j; ++k) d -= L_(j, k) * L_(j, k);
      if (!(d > 0.0)) ok_ = false;
      d = std::sqrt(d);
      L_(j, j) = d;
      for (Index i = j + 1; i < n; ++i) {
        double s = L_(i, j);
        for (Index k = 0; k < j; ++k) s -= L_(i, k) * L_(j, k);
        L_(i, j) = s / d;
      }
    }
  }
  template <class O>
  Matrix<double, R, 1> solve(const DenseBase<O>& b) const {
    const Index n = L_.rows();
    Matrix<double, R, 1> x(b.derived());
    for (Index i = 0; i < n; ++i) {
      double s = x[i];
      for (Index k = 0; k < i; ++k) s -= L_(i, k) * x[k];
      x[i] = s / L_(i, i);
    }
    for (Index i = n - 1; i >= 0; --i) {
      double s = x[i];
      for (Index k = i + 1; k < n; ++k) s -= L_(k, i) * x[k];
      x[i] = s / L_(i, i);
    }
    return x;
  }
  int info() const { return ok_ ? 0 : 1; }
};

// ---------------------------------------------------------------- array view
template <int R, int C>
struct ArrayWrap {
  double* d;
  Index r, c, rs, cs;
  ArrayWrap(double* d_, Index r_, Index c_, Index rs_, Index cs_) : d(d_), r(r_), c(c_), rs(rs_), cs(cs_) {}
  explicit ArrayWrap(const Result<R, C>& owned) : own(std::make_shared<Result<R, C>>(owned)) {
    d = own->data(); r = own->rows(); c = own->cols(); rs = 1; cs = r;
  }
  std::shared_ptr<Result<R, C>> own;
  double& at(Index i, Index j) const { return d[i * rs + j * cs]; }
  Index rows() const { return r; }
  Index cols() const { return c; }
  Index size() const { return r * c; }
  template <class F>
  ArrayWrap map(F f) const {
    Result<R, C> m(r, c, SizeTag{});
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) m.ref(i, j) = f(at(i, j));
    return ArrayWrap(m);
  }
  template <class F>
  ArrayWrap zip(const ArrayWrap& o, F f) const {
    internal::check(r == o.r && c == o.c, "array op: size mismatch");
    Result<R, C> m(r, c, SizeTag{});
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) m.ref(i, j) = f(at(i, j), o.at(i, j));
    return ArrayWrap(m);
  }
  template <class F>
  const ArrayWrap& update(const ArrayWrap& o, F f) const {
    const ArrayWrap src = o.map([](double v) { return v; });  // evaluate before writing
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) at(i, j) = f(at(i, j), src.at(i, j));
    return *this;
  }
  const ArrayWrap& operator*=(const ArrayWrap& o) const { return update(o, [](double a, double b) { return a * b; }); }
  const ArrayWrap& operator/=(const ArrayWrap& o) const { return update(o, [](double a, double b) { return a / b; }); }
  const ArrayWrap& operator+=(const ArrayWrap& o) const { return update(o, [](double a, double b) { return a + b; }); }
  const ArrayWrap& operator-=(const ArrayWrap& o) const { return update(o, [](double a, double b) { return a - b; }); }
  const ArrayWrap& operator*=(double s) const { for (Index k = 0; k < size(); ++k) at(k % r, k / r) *= s; return *this; }
  const ArrayWrap& operator/=(double s) const { for (Index k = 0; k < size(); ++k) at(k % r, k / r) /= s; return *this; }
  const ArrayWrap& operator+=(double s) const { for (Index k = 0; k < size(); ++k) at(k % r, k / r) += s; return *this; }
  const ArrayWrap& operator-=(double s) const { for (Index k = 0; k < size(); ++k) at(k % r, k / r) -= s; return *this; }
  ArrayWrap sqrt() const { return map([](double v) { return std::sqrt(v); }); }
  ArrayWrap square() const { return map([](double v) { return v * v; }); }
  ArrayWrap abs() const { return map([](double v) { return std::abs(v); }); }
  ArrayWrap exp() const { return map([](double v) { return std::exp(v); }); }
  ArrayWrap log() const { return map([](double v) { return std::log(v); }); }
  double sum() const {
    double s = 0.0;
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) s += at(i, j);
    return s;
  }
  Result<R, C> matrix() const {
    Result<R, C> m(r, c, SizeTag{});
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) m.ref(i, j) = at(i, j);
    return m;
  }
  operator Result<R, C>() const { return matrix(); }
};

template <int R, int C>
ArrayWrap<R, C> operator*(const ArrayWrap<R, C>& a, const ArrayWrap<R, C>& b) { return a.zip(b, [](double x, double y) { return x * y; }); }
template <int R, int C>
ArrayWrap<R, C> operator/(const ArrayWrap<R, C>& a, const ArrayWrap<R, C>& b) { return a.zip(b, [](double x, double y) { return x / y; }); }
template <int R, int C>
ArrayWrap<R, C> operator+(const ArrayWrap<R, C>& a, const ArrayWrap<R, C>& b) { return a.zip(b, [](double x, double y) { return x + y; }); }
template <int R, int C>
ArrayWrap<R, C> operator-(const ArrayWrap<R, C>& a, const ArrayWrap<R, C>& b) { return a.zip(b, [](double x, double y) { return x - y; }); }
template <int R, int C>
ArrayWrap<R, C> operator*(const ArrayWrap<R, C>& a, double s) { return a.map([s](double x) { return x * s; }); }
template <int R, int C>
ArrayWrap<R, C> operator*(double s, const ArrayWrap<R, C>& a) { return a.map([s](double x) { return s * x; }); }
template <int R, int C>
ArrayWrap<R, C> operator/(const ArrayWrap<R, C>& a, double s) { return a.map([s](double x) { return x / s; }); }
template <int R, int C>
ArrayWrap<R, C> operator/(double s, const ArrayWrap<R, C>& a) { return a.map([s](double x) { return s / x; }); }
template <int R, int C>
ArrayWrap<R, C> operator+(const ArrayWrap<R, C>& a, double s) { return a.map([s](double x) { return x + s; }); }
template <int R, int C>
ArrayWrap<R, C> operator-(const ArrayWrap<R, C>& a, double s) { return a.map([s](double x) { return x - s; }); }

// ---------------------------------------------------------------- arithmetic (eager)
template <class A, class B>
Result<internal::pick(A::Rows, B::Rows), internal::pick(A::Cols, B::Cols)> operator+(const DenseBase<A>& a,
                                                                                     const DenseBase<B>& b) {
  return a.binaryExpr(b, [](double x, double y) { return x + y; });
}
template <class A, class B>
Result<internal::pick(A::Rows, B::Rows), internal::pick(A::Cols, B::Cols)> operator-(const DenseBase<A>& a,
                                                                                     const DenseBase<B>& b) {
  return a.binaryExpr(b, [](double x, double y) { return x - y; });
}
template <class A>
Result<A::Rows, A::Cols> operator-(const DenseBase<A>& a) {
  return a.unaryExpr([](double x) { return -x; });
}
template <class A>
Result<A::Rows, A::Cols> operator*(const DenseBase<A>& a, double s) {
  return a.unaryExpr([s](double x) { return x * s; });
}
template <class A>
Result<A::Rows, A::Cols> operator*(double s, const DenseBase<A>& a) {
  return a.unaryExpr([s](double x) { return s * x; });
}
template <class A>
Result<A::Rows, A::Cols> operator/(const DenseBase<A>& a, double s) {
  return a.unaryExpr([s](double x) { return x / s; });
}
// matrix product: (i, j) = sum_k a(i, k) b(k, j), k ascending
template <class A, class B>
Result<A::Rows, B::Cols> operator*(const DenseBase<A>& a, const DenseBase<B>& b) {
  internal::check(a.cols() == b.rows(), "product: inner dimension mismatch");
  Result<A::Rows, B::Cols> r(a.rows(), b.cols(), SizeTag{});
  const Index K = a.cols();
  for (Index j = 0; j < b.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) {
      double s = 0.0;
      for (Index k = 0; k < K; ++k) s += a.coeff(i, k) * b.coeff(k, j);
      r.ref(i, j) = s;
    }
  return r;
}

using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using RowVectorXd = Matrix<double, 1, Dynamic>;
using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Vector4d = Matrix<double, 4, 1>;
using Matrix2d = Matrix<double, 2, 2>;
using Matrix3d = Matrix<double, 3, 3>;
template <class S, int N>
using Vector = Matrix<S, N, 1>;

}  // namespace Eigen
