// A minimal, eagerly evaluated restatement of the part of Eigen3's dense API
// that the reference sources on the hot path use, so those sources compile
// UNMODIFIED from /root/reference without Eigen being installed.
//
// TEST INFRASTRUCTURE ONLY.  This header exists to build oracle/_ref (the
// reference's own nn.cpp / nn_io.cpp / linalg.cpp and its doctest suites)
// as the parity checker.  Nothing in paper_2509_22462_b200/ includes it.
//
// Which third-party library this stands in for: Eigen3, "≥ 3.3", unpinned
// system package (proj/CMakeLists.txt:13, proj/README.md:40).  It is not
// vendored under /root/reference and not installed in this image or on the
// GPU box (probed: tools/probe_box.sh).  What is restated is Eigen's
// documented semantics for each member used, not its implementation:
//
//  * storage: column-major dense matrices (Eigen's default; linalg.hpp:10-11
//    aliases RealMat = MatrixXd, RealVec = VectorXd);
//  * expressions are evaluated eagerly into temporaries.  Eigen's lazy
//    evaluation changes only rounding order inside fused expressions, never
//    the value semantics; aliasing is always safe here (every assignment
//    goes through a fresh buffer), which is a superset of what .noalias()
//    promises;
//  * .array() switches to coefficient-wise semantics, .matrix() back;
//    rowwise()/colwise() broadcast a row / column vector;
//  * products go to the BLAS dgemm (EIGEN_USE_BLAS-style) when the build
//    defines GBOPT_REF_BLAS, else to a k-ordered triple loop;
//  * maxCoeff(&i) returns the FIRST index of the maximum (Eigen's
//    max_coeff_visitor updates only on a strictly greater value);
//  * comma initialisers fill row by row; PermutationMatrix P maps row i of
//    A to row indices(i) of P*A;
//  * HouseholderQR and SelfAdjointEigenSolver (used by the reference's
//    test_util.hpp / test_linalg.cpp only) are a textbook Householder QR and
//    a cyclic Jacobi eigenvalue iteration.
//
// Only double scalars are supported.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#ifdef GBOPT_REF_BLAS
extern "C" void scipy_cblas_dgemm64_(int order, int ta, int tb, std::int64_t m,
                                     std::int64_t n, std::int64_t k,
                                     double alpha, const double* a,
                                     std::int64_t lda, const double* b,
                                     std::int64_t ldb, double beta, double* c,
                                     std::int64_t ldc);
#endif

namespace Eigen {

using Index = std::ptrdiff_t;
enum { Dynamic = -1 };
enum UpLoType { Lower = 1, Upper = 2 };
enum { Infinity = -1 };

template <typename S, int R, int C, int O = 0, int MR = R, int MC = C>
class Matrix;
class MatView;
class ArrView;
class ArrayXX;

namespace internal {

[[noreturn]] inline void fail(const char* what) {
  throw std::logic_error(std::string("eigen_subset: ") + what);
}

// A strided column-major window: element (i, j) lives at p[i*rs + j*cs].
struct Dense {
  double* p_ = nullptr;
  Index r_ = 0, c_ = 0, rs_ = 1, cs_ = 0;

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double& at(Index i, Index j) const { return p_[i * rs_ + j * cs_]; }
  bool is_vector() const { return r_ == 1 || c_ == 1; }
  // Linear (vector or column-major) element k.
  double& lin(Index k) const {
    if (c_ == 1) return p_[k * rs_];
    if (r_ == 1) return p_[k * cs_];
    return p_[(k % r_) * rs_ + (k / r_) * cs_];
  }
};

struct MatTag {};
struct ArrTag {};

template <class T>
constexpr bool is_dense_v = std::is_base_of_v<Dense, std::decay_t<T>>;
template <class T>
constexpr bool is_mat_v = std::is_base_of_v<MatTag, std::decay_t<T>>;
template <class T>
constexpr bool is_arr_v = std::is_base_of_v<ArrTag, std::decay_t<T>>;

// std::vector whose resize() leaves doubles uninitialised (producers write
// every element; alloc() below zero-fills explicitly where Eigen semantics
// need it).
template <class T>
struct UninitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = UninitAlloc<U>;
  };
  UninitAlloc() = default;
  template <class U>
  UninitAlloc(const UninitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept { ::new (static_cast<void*>(p)) U; }
  template <class U, class... A>
  void construct(U* p, A&&... a) { ::new (static_cast<void*>(p)) U(std::forward<A>(a)...); }
};
using Buffer = std::vector<double, UninitAlloc<double>>;

inline bool contiguous(const Dense& d) {
  return d.size() == 0 || (d.rs_ == 1 && (d.cs_ == d.r_ || d.c_ == 1)) || (d.r_ == 1 && d.c_ == 1);
}
inline bool overlap(const Dense& a, const Dense& b) {
  if (a.size() == 0 || b.size() == 0) return false;
  const double* a0 = a.p_;
  const double* a1 = a.p_ + (a.r_ - 1) * a.rs_ + (a.c_ - 1) * a.cs_;
  const double* b0 = b.p_;
  const double* b1 = b.p_ + (b.r_ - 1) * b.rs_ + (b.c_ - 1) * b.cs_;
  return !(a1 < b0 || b1 < a0);
}

inline Buffer snapshot(const Dense& d) {
  Buffer v(static_cast<size_t>(d.size()));
  if (contiguous(d) && d.size() > 0) {
    std::memcpy(v.data(), d.p_, sizeof(double) * static_cast<size_t>(d.size()));
    return v;
  }
  for (Index j = 0; j < d.c_; ++j)
    for (Index i = 0; i < d.r_; ++i) v[static_cast<size_t>(i + j * d.r_)] = d.at(i, j);
  return v;
}

// Writes src into dst elementwise (shapes must agree; vectors of either
// orientation may be assigned to each other, as Eigen allows).
inline void copy_into(const Dense& dst, const Dense& src) {
  if (dst.size() != src.size()) fail("assignment size mismatch");
  const bool same = dst.r_ == src.r_ && dst.c_ == src.c_;
  if (!same && !(dst.is_vector() && src.is_vector())) fail("assignment shape mismatch");
  if (!overlap(dst, src)) {
    if (same) {
      for (Index j = 0; j < dst.c_; ++j)
        for (Index i = 0; i < dst.r_; ++i) dst.at(i, j) = src.at(i, j);
    } else {
      for (Index k = 0; k < dst.size(); ++k) dst.lin(k) = src.lin(k);
    }
    return;
  }
  const Buffer tmp = snapshot(src);
  if (same) {
    for (Index j = 0; j < dst.c_; ++j)
      for (Index i = 0; i < dst.r_; ++i) dst.at(i, j) = tmp[static_cast<size_t>(i + j * dst.r_)];
  } else {
    for (Index k = 0; k < dst.size(); ++k) dst.lin(k) = tmp[static_cast<size_t>(k)];
  }
}

template <class F>
inline void for_each(const Dense& d, F&& f) {
  for (Index j = 0; j < d.c_; ++j)
    for (Index i = 0; i < d.r_; ++i) f(d.at(i, j), i, j);
}

inline void check_same(const Dense& a, const Dense& b) {
  if (a.r_ != b.r_ || a.c_ != b.c_) {
    if (!(a.is_vector() && b.is_vector() && a.size() == b.size()))
      fail("coefficient-wise operands differ in shape");
  }
}

// Column-major descriptor for BLAS; false if the window needs a copy.
inline bool blas_desc(const Dense& d, int& trans, Index& ld) {
  const int kNo = 111, kT = 112;
  if (d.r_ == 1 && d.c_ == 1) { trans = kNo; ld = 1; return true; }
  if (d.c_ == 1) {
    if (d.rs_ == 1) { trans = kNo; ld = std::max<Index>(d.r_, 1); return true; }
    trans = kT; ld = d.rs_; return d.rs_ >= 1;
  }
  if (d.r_ == 1) { trans = kNo; ld = d.cs_; return d.cs_ >= 1; }
  if (d.rs_ == 1 && d.cs_ >= d.r_) { trans = kNo; ld = d.cs_; return true; }
  if (d.cs_ == 1 && d.rs_ >= d.c_) { trans = kT; ld = d.rs_; return true; }
  return false;
}

}  // namespace internal

using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using RowVectorXd = Matrix<double, 1, Dynamic>;
using ArrayXd = ArrayXX;
using ArrayXXd = ArrayXX;

// ---------------------------------------------------------------- broadcasts
class ArrView;
struct Broadcast {
  internal::Dense t;
  bool colwise;  // true: vector runs down each column (length rows)
  double vec_at(const internal::Dense& v, Index i, Index j) const {
    return v.lin(colwise ? i : j);
  }
  void check(const internal::Dense& v) const {
    if (v.size() != (colwise ? t.r_ : t.c_)) internal::fail("broadcast length mismatch");
  }
  template <class V> ArrayXX operator*(const V& v) const;
  template <class V> ArrayXX operator/(const V& v) const;
  template <class V> ArrayXX operator+(const V& v) const;
  template <class V> ArrayXX operator-(const V& v) const;
  template <class V> void operator*=(const V& v) const {
    check(v);
    internal::for_each(t, [&](double& x, Index i, Index j) { x *= vec_at(v, i, j); });
  }
  template <class V> void operator/=(const V& v) const {
    check(v);
    internal::for_each(t, [&](double& x, Index i, Index j) { x /= vec_at(v, i, j); });
  }
  template <class V> void operator+=(const V& v) const {
    check(v);
    internal::for_each(t, [&](double& x, Index i, Index j) { x += vec_at(v, i, j); });
  }
  template <class V> void operator-=(const V& v) const {
    check(v);
    internal::for_each(t, [&](double& x, Index i, Index j) { x -= vec_at(v, i, j); });
  }
};

template <int UpLo>
struct SelfAdjointView {
  internal::Dense a;
};

// ------------------------------------------------------- shared member set
template <class Derived>
class CommonOps {
 protected:
  const internal::Dense& d() const { return static_cast<const Derived&>(*this); }

 public:
  MatrixXd cwiseAbs() const;
  template <class O> MatrixXd cwiseProduct(const O& o) const;
  double maxCoeff() const {
    if (d().size() == 0) internal::fail("maxCoeff of an empty object");
    double m = d().lin(0);
    for (Index k = 1; k < d().size(); ++k) if (d().lin(k) > m) m = d().lin(k);
    return m;
  }
  double maxCoeff(Index* idx) const {
    if (d().size() == 0) internal::fail("maxCoeff of an empty object");
    double m = d().lin(0);
    Index best = 0;
    for (Index k = 1; k < d().size(); ++k)
      if (d().lin(k) > m) { m = d().lin(k); best = k; }
    if (idx) *idx = best;
    return m;
  }
  double minCoeff() const {
    if (d().size() == 0) internal::fail("minCoeff of an empty object");
    double m = d().lin(0);
    for (Index k = 1; k < d().size(); ++k) if (d().lin(k) < m) m = d().lin(k);
    return m;
  }
  double sum() const {
    double s = 0.0;
    internal::for_each(d(), [&](double& x, Index, Index) { s += x; });
    return s;
  }
  template <class O> double dot(const O& o) const {
    if (d().size() != o.size()) internal::fail("dot size mismatch");
    double s = 0.0;
    for (Index k = 0; k < d().size(); ++k) s += d().lin(k) * o.lin(k);
    return s;
  }
  bool allFinite() const {
    bool ok = true;
    internal::for_each(d(), [&](double& x, Index, Index) { ok = ok && std::isfinite(x); });
    return ok;
  }
  template <int P> double lpNorm() const {
    static_assert(P == Infinity, "eigen_subset: only lpNorm<Infinity>");
    double m = 0.0;
    internal::for_each(d(), [&](double& x, Index, Index) { m = std::max(m, std::abs(x)); });
    return m;
  }
  double norm() const {
    double s = 0.0;
    internal::for_each(d(), [&](double& x, Index, Index) { s += x * x; });
    return std::sqrt(s);
  }
  double& operator()(Index i, Index j) const { return d().at(i, j); }
  double& operator()(Index k) const { return d().lin(k); }
  double& operator[](Index k) const { return d().lin(k); }
  double& coeffRef(Index i, Index j) const { return d().at(i, j); }
  double coeff(Index i, Index j) const { return d().at(i, j); }
  double& coeffRef(Index k) const { return d().lin(k); }
  double coeff(Index k) const { return d().lin(k); }
};

// ------------------------------------------------- matrix-semantics members
template <class Derived>
class MatOps : public CommonOps<Derived>, public internal::MatTag {
  using CommonOps<Derived>::d;

 public:
  MatView block(Index i, Index j, Index h, Index w) const;
  MatView col(Index j) const;
  MatView row(Index i) const;
  MatView segment(Index i, Index n) const;
  MatView head(Index n) const;
  MatView tail(Index n) const;
  MatView diagonal() const;
  MatView transpose() const;
  MatView topRows(Index n) const;
  MatView leftCols(Index n) const;
  ArrView array() const;
  MatrixXd asDiagonal() const;
  template <int UpLo> SelfAdjointView<UpLo> selfadjointView() const {
    return SelfAdjointView<UpLo>{d()};
  }
  template <int UpLo> MatrixXd triangularView() const;
  const Derived& matrix() const { return static_cast<const Derived&>(*this); }
  MatrixXd eval() const;
};

// --------------------------------------------------------------- views
class MatView : public internal::Dense, public MatOps<MatView> {
 public:
  MatView() = default;
  explicit MatView(const internal::Dense& d) : internal::Dense(d) {}
  MatView(const MatView&) = default;
  // Assignment writes through (a view never rebinds).
  MatView& operator=(const MatView& o) { internal::copy_into(*this, o); return *this; }
  template <class T, std::enable_if_t<internal::is_dense_v<T>, int> = 0>
  MatView& operator=(const T& o) { internal::copy_into(*this, o); return *this; }
  template <class T, std::enable_if_t<internal::is_dense_v<T>, int> = 0>
  const MatView& operator+=(const T& o) const;
  template <class T, std::enable_if_t<internal::is_dense_v<T>, int> = 0>
  const MatView& operator-=(const T& o) const;
  const MatView& operator*=(double s) const {
    internal::for_each(*this, [&](double& x, Index, Index) { x *= s; });
    return *this;
  }
  const MatView& operator/=(double s) const {
    internal::for_each(*this, [&](double& x, Index, Index) { x /= s; });
    return *this;
  }
  MatView noalias() const { return *this; }
  void setZero() const { internal::for_each(*this, [](double& x, Index, Index) { x = 0.0; }); }
  void setConstant(double v) const { internal::for_each(*this, [&](double& x, Index, Index) { x = v; }); }
  void swap(MatView o) const {
    if (o.r_ != r_ || o.c_ != c_) internal::fail("swap shape mismatch");
    internal::for_each(*this, [&](double& x, Index i, Index j) { std::swap(x, o.at(i, j)); });
  }
};

class ArrView : public internal::Dense, public CommonOps<ArrView>, public internal::ArrTag {
 public:
  ArrView() = default;
  explicit ArrView(const internal::Dense& d) : internal::Dense(d) {}
  ArrView(const ArrView&) = default;
  ArrView& operator=(const ArrView& o) { internal::copy_into(*this, o); return *this; }
  template <class T, std::enable_if_t<internal::is_dense_v<T>, int> = 0>
  ArrView& operator=(const T& o) { internal::copy_into(*this, o); return *this; }
  Broadcast colwise() const { return Broadcast{*this, true}; }
  Broadcast rowwise() const { return Broadcast{*this, false}; }
  MatView matrix() const { return MatView(*this); }
  ArrayXX exp() const;
  ArrayXX tanh() const;
  ArrayXX square() const;
  ArrayXX abs() const;
  ArrayXX log() const;
  ArrayXX sqrt() const;
  const ArrView& operator*=(double s) const {
    internal::for_each(*this, [&](double& x, Index, Index) { x *= s; });
    return *this;
  }
  template <class T, std::enable_if_t<internal::is_arr_v<T>, int> = 0>
  const ArrView& operator*=(const T& o) const {
    internal::check_same(*this, o);
    const internal::Buffer tmp = internal::snapshot(o);
    internal::for_each(*this, [&](double& x, Index i, Index j) { x *= tmp[static_cast<size_t>(i + j * r_)]; });
    return *this;
  }
  template <class T, std::enable_if_t<internal::is_arr_v<T>, int> = 0>
  const ArrView& operator/=(const T& o) const {
    internal::check_same(*this, o);
    const internal::Buffer tmp = internal::snapshot(o);
    internal::for_each(*this, [&](double& x, Index i, Index j) { x /= tmp[static_cast<size_t>(i + j * r_)]; });
    return *this;
  }
};

// --------------------------------------------------------------- owners
namespace internal {
template <class Self>
struct Owned : Dense {
  Buffer buf_;
  void rebind(Index r, Index c) {
    r_ = r; c_ = c; rs_ = 1; cs_ = r;
    p_ = buf_.empty() ? nullptr : buf_.data();
  }
  void alloc(Index r, Index c) {
    if (r < 0 || c < 0) fail("negative dimension");
    buf_.assign(static_cast<size_t>(r * c), 0.0);
    rebind(r, c);
  }
  void alloc_uninit(Index r, Index c) {
    if (r < 0 || c < 0) fail("negative dimension");
    buf_.clear();
    buf_.resize(static_cast<size_t>(r * c));
    rebind(r, c);
  }
  void take(Buffer&& v, Index r, Index c) {
    buf_ = std::move(v);
    rebind(r, c);
  }
};
}  // namespace internal

class ArrayXX : public internal::Owned<ArrayXX>, public CommonOps<ArrayXX>, public internal::ArrTag {
 public:
  ArrayXX() { rebind(0, 0); }
  ArrayXX(Index r, Index c) { alloc(r, c); }
  ArrayXX(const ArrayXX& o) { buf_ = o.buf_; rebind(o.r_, o.c_); }
  template <int R, int C, int O, int MR, int MC>
  ArrayXX(Matrix<double, R, C, O, MR, MC>&& o) {
    const Index r = o.r_, c = o.c_;
    take(std::move(o.buf_), r, c);
    o.buf_.clear();
    o.rebind(0, 0);
  }
  ArrayXX(ArrayXX&& o) noexcept { buf_ = std::move(o.buf_); rebind(o.r_, o.c_); o.rebind(0, 0); }
  template <class T, std::enable_if_t<internal::is_dense_v<T> && !std::is_same_v<std::decay_t<T>, ArrayXX>, int> = 0>
  ArrayXX(const T& src) { take(internal::snapshot(src), src.rows(), src.cols()); }
  ArrayXX& operator=(const ArrayXX& o) { internal::Buffer v = o.buf_; take(std::move(v), o.r_, o.c_); return *this; }
  ArrayXX& operator=(ArrayXX&& o) noexcept { buf_ = std::move(o.buf_); rebind(o.r_, o.c_); o.rebind(0, 0); return *this; }
  template <class T, std::enable_if_t<internal::is_dense_v<T> && !std::is_same_v<std::decay_t<T>, ArrayXX>, int> = 0>
  ArrayXX& operator=(const T& src) { take(internal::snapshot(src), src.rows(), src.cols()); return *this; }
  ArrView view() const { return ArrView(*this); }
  Broadcast colwise() const { return Broadcast{*this, true}; }
  Broadcast rowwise() const { return Broadcast{*this, false}; }
  MatView matrix() const& { return MatView(*this); }
  MatrixXd matrix() &&;
  ArrayXX exp() const { return view().exp(); }
  ArrayXX tanh() const { return view().tanh(); }
  ArrayXX square() const { return view().square(); }
  ArrayXX abs() const { return view().abs(); }
  ArrayXX log() const { return view().log(); }
  ArrayXX sqrt() const { return view().sqrt(); }
};

template <typename S, int R, int C, int O, int MR, int MC>
class Matrix : public internal::Owned<Matrix<S, R, C, O, MR, MC>>,
               public MatOps<Matrix<S, R, C, O, MR, MC>> {
  static_assert(std::is_same_v<S, double>, "eigen_subset: double only");
  using Base = internal::Owned<Matrix<S, R, C, O, MR, MC>>;

 public:
  using Base::alloc;
  using Base::alloc_uninit;
  using Base::rebind;
  using Base::take;
  using Base::buf_;

 private:

  static constexpr bool kCol = (C == 1);
  static constexpr bool kRow = (R == 1);

  // Shape an incoming object takes inside this type (vectors keep their
  // compile-time orientation).
  static void target_shape(const internal::Dense& src, Index& r, Index& c) {
    if (kCol) {
      if (!src.is_vector() && src.size() != 0) internal::fail("matrix assigned to a column vector");
      r = src.size(); c = 1;
    } else if (kRow) {
      if (!src.is_vector() && src.size() != 0) internal::fail("matrix assigned to a row vector");
      r = 1; c = src.size();
    } else {
      r = src.r_; c = src.c_;
    }
  }
  void assign(const internal::Dense& src) {
    Index r, c;
    target_shape(src, r, c);
    if (internal::contiguous(src) && !internal::overlap(*this, src)) {
      internal::Buffer v(static_cast<size_t>(r * c));
      if (r * c > 0) std::memcpy(v.data(), src.p_, sizeof(double) * static_cast<size_t>(r * c));
      take(std::move(v), r, c);
      return;
    }
    internal::Buffer v(static_cast<size_t>(r * c));
    if (r == src.r_ && c == src.c_) {
      for (Index j = 0; j < c; ++j)
        for (Index i = 0; i < r; ++i) v[static_cast<size_t>(i + j * r)] = src.at(i, j);
    } else {
      for (Index k = 0; k < r * c; ++k) v[static_cast<size_t>(k)] = src.lin(k);
    }
    take(std::move(v), r, c);
  }

 public:
  using internal::Dense::cols;
  using internal::Dense::rows;
  using internal::Dense::size;

  Matrix() { rebind(kCol ? 0 : (kRow ? 1 : 0), kRow ? 0 : (kCol ? 1 : 0)); }
  explicit Matrix(Index n) {
    static_assert(kCol || kRow, "eigen_subset: Matrix(n) needs a vector type");
    alloc(kCol ? n : 1, kCol ? 1 : n);
  }
  Matrix(Index r, Index c) { alloc(r, c); }
  Matrix(const Matrix& o) { buf_ = o.buf_; rebind(o.r_, o.c_); }
  Matrix(Matrix&& o) noexcept { buf_ = std::move(o.buf_); rebind(o.r_, o.c_); o.buf_.clear(); o.rebind(kRow ? 1 : 0, kCol ? 1 : 0); }
  template <class T, std::enable_if_t<internal::is_dense_v<T> && !std::is_same_v<std::decay_t<T>, Matrix>, int> = 0>
  Matrix(const T& src) { assign(src); }
  // Steal the buffer of another owner (same column-major layout).
  template <int R2, int C2, int O2, int MR2, int MC2,
            std::enable_if_t<!(R2 == R && C2 == C && O2 == O && MR2 == MR && MC2 == MC), int> = 0>
  Matrix(Matrix<S, R2, C2, O2, MR2, MC2>&& o) { steal(o); }
  Matrix(ArrayXX&& o);
  template <int R2, int C2, int O2, int MR2, int MC2,
            std::enable_if_t<!(R2 == R && C2 == C && O2 == O && MR2 == MR && MC2 == MC), int> = 0>
  Matrix& operator=(Matrix<S, R2, C2, O2, MR2, MC2>&& o) { steal(o); return *this; }
  Matrix& operator=(ArrayXX&& o);
  template <class Own>
  void steal(Own& o) {
    Index r, c;
    target_shape(o, r, c);
    take(std::move(o.buf_), r, c);
    o.buf_.clear();
    o.rebind(0, 0);
  }

  Matrix& operator=(const Matrix& o) { if (this != &o) assign(o); return *this; }
  Matrix& operator=(Matrix&& o) noexcept {
    buf_ = std::move(o.buf_); rebind(o.r_, o.c_);
    o.buf_.clear(); o.rebind(kRow ? 1 : 0, kCol ? 1 : 0);
    return *this;
  }
  template <class T, std::enable_if_t<internal::is_dense_v<T> && !std::is_same_v<std::decay_t<T>, Matrix>, int> = 0>
  Matrix& operator=(const T& src) { assign(src); return *this; }

  template <class T, std::enable_if_t<internal::is_dense_v<T>, int> = 0>
  Matrix& operator+=(const T& o) { MatView(*this) += o; return *this; }
  template <class T, std::enable_if_t<internal::is_dense_v<T>, int> = 0>
  Matrix& operator-=(const T& o) { MatView(*this) -= o; return *this; }
  Matrix& operator*=(double s) { MatView(*this) *= s; return *this; }
  Matrix& operator/=(double s) { MatView(*this) /= s; return *this; }
  Matrix& noalias() { return *this; }

  void resize(Index n) {
    static_assert(kCol || kRow, "eigen_subset: resize(n) needs a vector type");
    alloc(kCol ? n : 1, kCol ? 1 : n);
  }
  void resize(Index r, Index c) { alloc(r, c); }
  void setZero() { MatView(*this).setZero(); }
  void swap(MatView o) { MatView(*this).swap(o); }
  double* data() { return buf_.data(); }
  const double* data() const { return buf_.data(); }

  static Matrix Zero(Index n) { return Matrix(n); }
  static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
  static Matrix Constant(Index n, double v) { Matrix m(n); m.setConstantAll(v); return m; }
  static Matrix Constant(Index r, Index c, double v) { Matrix m(r, c); m.setConstantAll(v); return m; }
  static Matrix Ones(Index n) { return Constant(n, 1.0); }
  static Matrix Ones(Index r, Index c) { return Constant(r, c, 1.0); }
  static Matrix Identity(Index r, Index c) {
    Matrix m(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m.at(i, i) = 1.0;
    return m;
  }

  // Comma initialiser: fills row by row.
  struct CommaInit {
    Matrix* m;
    Index k;
    CommaInit& operator,(double v) { put(v); return *this; }
    void put(double v) {
      if (k >= m->size()) internal::fail("too many coefficients in comma initialiser");
      const Index i = k / m->c_, j = k % m->c_;
      m->at(i, j) = v;
      ++k;
    }
  };
  CommaInit operator<<(double v) { CommaInit ci{this, 0}; ci.put(v); return ci; }

 private:
  void setConstantAll(double v) { std::fill(buf_.begin(), buf_.end(), v); }
};

template <typename S, int R, int C, int O, int MR, int MC>
Matrix<S, R, C, O, MR, MC>::Matrix(ArrayXX&& o) { steal(o); }
template <typename S, int R, int C, int O, int MR, int MC>
Matrix<S, R, C, O, MR, MC>& Matrix<S, R, C, O, MR, MC>::operator=(ArrayXX&& o) { steal(o); return *this; }
inline MatrixXd ArrayXX::matrix() && { return MatrixXd(std::move(*this)); }

// ----------------------------------------------------- member definitions
template <class D> MatView MatOps<D>::block(Index i, Index j, Index h, Index w) const {
  const internal::Dense& s = d();
  if (i < 0 || j < 0 || h < 0 || w < 0 || i + h > s.r_ || j + w > s.c_) internal::fail("block out of range");
  internal::Dense v{s.p_ + i * s.rs_ + j * s.cs_, h, w, s.rs_, s.cs_};
  return MatView(v);
}
template <class D> MatView MatOps<D>::col(Index j) const { return block(0, j, d().r_, 1); }
template <class D> MatView MatOps<D>::row(Index i) const { return block(i, 0, 1, d().c_); }
template <class D> MatView MatOps<D>::segment(Index i, Index n) const {
  const internal::Dense& s = d();
  if (!s.is_vector()) internal::fail("segment of a matrix");
  return s.c_ == 1 ? block(i, 0, n, 1) : block(0, i, 1, n);
}
template <class D> MatView MatOps<D>::head(Index n) const { return segment(0, n); }
template <class D> MatView MatOps<D>::tail(Index n) const { return segment(d().size() - n, n); }
template <class D> MatView MatOps<D>::topRows(Index n) const { return block(0, 0, n, d().c_); }
template <class D> MatView MatOps<D>::leftCols(Index n) const { return block(0, 0, d().r_, n); }
template <class D> MatView MatOps<D>::diagonal() const {
  const internal::Dense& s = d();
  internal::Dense v{s.p_, std::min(s.r_, s.c_), 1, s.rs_ + s.cs_, 0};
  return MatView(v);
}
template <class D> MatView MatOps<D>::transpose() const {
  const internal::Dense& s = d();
  internal::Dense v{s.p_, s.c_, s.r_, s.cs_, s.rs_};
  return MatView(v);
}
template <class D> ArrView MatOps<D>::array() const { return ArrView(d()); }
template <class D> MatrixXd MatOps<D>::eval() const { return MatrixXd(d()); }
template <class D> MatrixXd MatOps<D>::asDiagonal() const {
  const internal::Dense& s = d();
  if (!s.is_vector()) internal::fail("asDiagonal of a matrix");
  MatrixXd m(s.size(), s.size());
  for (Index k = 0; k < s.size(); ++k) m(k, k) = s.lin(k);
  return m;
}
template <class D> template <int UpLo> MatrixXd MatOps<D>::triangularView() const {
  MatrixXd m(d());
  for (Index j = 0; j < m.cols(); ++j)
    for (Index i = 0; i < m.rows(); ++i)
      if ((UpLo == Upper && i > j) || (UpLo == Lower && i < j)) m(i, j) = 0.0;
  return m;
}
template <class D> MatrixXd CommonOps<D>::cwiseAbs() const {
  MatrixXd m(d());
  internal::for_each(m, [](double& x, Index, Index) { x = std::abs(x); });
  return m;
}
template <class D> template <class O> MatrixXd CommonOps<D>::cwiseProduct(const O& o) const {
  internal::check_same(d(), o);
  MatrixXd m(d());
  for (Index k = 0; k < m.size(); ++k) m.lin(k) *= o.lin(k);
  return m;
}

// ------------------------------------------------------------- products
namespace internal {
inline MatrixXd product(const Dense& a, const Dense& b) {
  if (a.c_ != b.r_) fail("product inner dimensions differ");
  MatrixXd c(a.r_, b.c_);
  if (a.r_ == 0 || b.c_ == 0) return c;
  if (a.c_ == 0) return c;
#ifdef GBOPT_REF_BLAS
  int ta, tb;
  Index lda, ldb;
  MatrixXd ca, cb;
  const Dense* pa = &a;
  const Dense* pb = &b;
  if (!blas_desc(*pa, ta, lda)) { ca = MatrixXd(a); pa = &ca; blas_desc(*pa, ta, lda); }
  if (!blas_desc(*pb, tb, ldb)) { cb = MatrixXd(b); pb = &cb; blas_desc(*pb, tb, ldb); }
  scipy_cblas_dgemm64_(102, ta, tb, a.r_, b.c_, a.c_, 1.0, pa->p_, lda, pb->p_, ldb, 0.0,
                       c.data(), a.r_);
#else
  for (Index j = 0; j < b.c_; ++j)
    for (Index k = 0; k < a.c_; ++k) {
      const double bkj = b.at(k, j);
      for (Index i = 0; i < a.r_; ++i) c.at(i, j) += a.at(i, k) * bkj;
    }
#endif
  return c;
}

template <class F>
inline MatrixXd map2(const Dense& a, const Dense& b, F f) {
  check_same(a, b);
  MatrixXd m;
  m.alloc_uninit(a.r_, a.c_);
  double* o = m.data();
  const Index n = a.size();
  if (contiguous(a) && contiguous(b)) {
    for (Index k = 0; k < n; ++k) o[k] = f(a.p_[k], b.p_[k]);
  } else if (a.r_ == b.r_ && a.c_ == b.c_) {
    for (Index j = 0; j < a.c_; ++j)
      for (Index i = 0; i < a.r_; ++i) o[i + j * a.r_] = f(a.at(i, j), b.at(i, j));
  } else {
    for (Index k = 0; k < n; ++k) o[k] = f(a.lin(k), b.lin(k));
  }
  return m;
}
template <class F>
inline MatrixXd map1(const Dense& a, F f) {
  MatrixXd m;
  m.alloc_uninit(a.r_, a.c_);
  double* o = m.data();
  if (contiguous(a)) {
    for (Index k = 0; k < a.size(); ++k) o[k] = f(a.p_[k]);
  } else {
    for (Index j = 0; j < a.c_; ++j)
      for (Index i = 0; i < a.r_; ++i) o[i + j * a.r_] = f(a.at(i, j));
  }
  return m;
}
}  // namespace internal

template <class T, std::enable_if_t<internal::is_dense_v<T>, int>>
const MatView& MatView::operator+=(const T& o) const {
  internal::check_same(*this, o);
  if (!internal::overlap(*this, o)) {
    if (r_ == o.rows() && c_ == o.cols()) {
      internal::for_each(*this, [&](double& x, Index i, Index j) { x += o.at(i, j); });
    } else {
      for (Index k = 0; k < size(); ++k) lin(k) += o.lin(k);
    }
    return *this;
  }
  const internal::Buffer tmp = internal::snapshot(o);
  if (r_ == o.rows() && c_ == o.cols()) {
    internal::for_each(*this, [&](double& x, Index i, Index j) { x += tmp[static_cast<size_t>(i + j * r_)]; });
  } else {
    for (Index k = 0; k < size(); ++k) lin(k) += tmp[static_cast<size_t>(k)];
  }
  return *this;
}
template <class T, std::enable_if_t<internal::is_dense_v<T>, int>>
const MatView& MatView::operator-=(const T& o) const {
  internal::check_same(*this, o);
  if (!internal::overlap(*this, o)) {
    if (r_ == o.rows() && c_ == o.cols()) {
      internal::for_each(*this, [&](double& x, Index i, Index j) { x -= o.at(i, j); });
    } else {
      for (Index k = 0; k < size(); ++k) lin(k) -= o.lin(k);
    }
    return *this;
  }
  const internal::Buffer tmp = internal::snapshot(o);
  if (r_ == o.rows() && c_ == o.cols()) {
    internal::for_each(*this, [&](double& x, Index i, Index j) { x -= tmp[static_cast<size_t>(i + j * r_)]; });
  } else {
    for (Index k = 0; k < size(); ++k) lin(k) -= tmp[static_cast<size_t>(k)];
  }
  return *this;
}

inline ArrayXX ArrView::exp() const { return ArrayXX(internal::map1(*this, [](double x) { return std::exp(x); })); }
inline ArrayXX ArrView::tanh() const { return ArrayXX(internal::map1(*this, [](double x) { return std::tanh(x); })); }
inline ArrayXX ArrView::square() const { return ArrayXX(internal::map1(*this, [](double x) { return x * x; })); }
inline ArrayXX ArrView::abs() const { return ArrayXX(internal::map1(*this, [](double x) { return std::abs(x); })); }
inline ArrayXX ArrView::log() const { return ArrayXX(internal::map1(*this, [](double x) { return std::log(x); })); }
inline ArrayXX ArrView::sqrt() const { return ArrayXX(internal::map1(*this, [](double x) { return std::sqrt(x); })); }

template <class V> ArrayXX Broadcast::operator*(const V& v) const {
  check(v);
  ArrayXX out;
  out.alloc_uninit(t.r_, t.c_);
  double* o = out.buf_.data();
  if (colwise) {
    const internal::Buffer vv = internal::snapshot(v);
    for (Index j = 0; j < t.c_; ++j)
      for (Index i = 0; i < t.r_; ++i) o[i + j * t.r_] = t.at(i, j) * vv[static_cast<size_t>(i)];
  } else {
    for (Index j = 0; j < t.c_; ++j) {
      const double s = v.lin(j);
      for (Index i = 0; i < t.r_; ++i) o[i + j * t.r_] = t.at(i, j) * s;
    }
  }
  return out;
}
template <class V> ArrayXX Broadcast::operator/(const V& v) const {
  check(v);
  ArrayXX out;
  out.alloc_uninit(t.r_, t.c_);
  double* o = out.buf_.data();
  if (colwise) {
    const internal::Buffer vv = internal::snapshot(v);
    for (Index j = 0; j < t.c_; ++j)
      for (Index i = 0; i < t.r_; ++i) o[i + j * t.r_] = t.at(i, j) / vv[static_cast<size_t>(i)];
  } else {
    for (Index j = 0; j < t.c_; ++j) {
      const double s = v.lin(j);
      for (Index i = 0; i < t.r_; ++i) o[i + j * t.r_] = t.at(i, j) / s;
    }
  }
  return out;
}
template <class V> ArrayXX Broadcast::operator+(const V& v) const {
  check(v);
  ArrayXX out;
  out.alloc_uninit(t.r_, t.c_);
  double* o = out.buf_.data();
  if (colwise) {
    const internal::Buffer vv = internal::snapshot(v);
    for (Index j = 0; j < t.c_; ++j)
      for (Index i = 0; i < t.r_; ++i) o[i + j * t.r_] = t.at(i, j) + vv[static_cast<size_t>(i)];
  } else {
    for (Index j = 0; j < t.c_; ++j) {
      const double s = v.lin(j);
      for (Index i = 0; i < t.r_; ++i) o[i + j * t.r_] = t.at(i, j) + s;
    }
  }
  return out;
}
template <class V> ArrayXX Broadcast::operator-(const V& v) const {
  check(v);
  ArrayXX out;
  out.alloc_uninit(t.r_, t.c_);
  double* o = out.buf_.data();
  if (colwise) {
    const internal::Buffer vv = internal::snapshot(v);
    for (Index j = 0; j < t.c_; ++j)
      for (Index i = 0; i < t.r_; ++i) o[i + j * t.r_] = t.at(i, j) - vv[static_cast<size_t>(i)];
  } else {
    for (Index j = 0; j < t.c_; ++j) {
      const double s = v.lin(j);
      for (Index i = 0; i < t.r_; ++i) o[i + j * t.r_] = t.at(i, j) - s;
    }
  }
  return out;
}

// ------------------------------------------------------------- operators
// Matrix semantics: * is the matrix product.
template <class A, class B, std::enable_if_t<internal::is_mat_v<A> && internal::is_mat_v<B>, int> = 0>
MatrixXd operator*(const A& a, const B& b) { return internal::product(a, b); }
template <class A, class B, std::enable_if_t<internal::is_mat_v<A> && internal::is_mat_v<B>, int> = 0>
MatrixXd operator+(const A& a, const B& b) { return internal::map2(a, b, [](double x, double y) { return x + y; }); }
template <class A, class B, std::enable_if_t<internal::is_mat_v<A> && internal::is_mat_v<B>, int> = 0>
MatrixXd operator-(const A& a, const B& b) { return internal::map2(a, b, [](double x, double y) { return x - y; }); }
template <class A, std::enable_if_t<internal::is_mat_v<A>, int> = 0>
MatrixXd operator-(const A& a) { return internal::map1(a, [](double x) { return -x; }); }
template <class A, std::enable_if_t<internal::is_mat_v<A>, int> = 0>
MatrixXd operator*(const A& a, double s) { return internal::map1(a, [s](double x) { return x * s; }); }
template <class A, std::enable_if_t<internal::is_mat_v<A>, int> = 0>
MatrixXd operator*(double s, const A& a) { return internal::map1(a, [s](double x) { return s * x; }); }
template <class A, std::enable_if_t<internal::is_mat_v<A>, int> = 0>
MatrixXd operator/(const A& a, double s) { return internal::map1(a, [s](double x) { return x / s; }); }

// Array semantics: coefficient-wise.
#define GBOPT_SUBSET_ARR_BINOP(OP)                                                          \
  template <class A, class B,                                                               \
            std::enable_if_t<internal::is_arr_v<A> && internal::is_arr_v<B>, int> = 0>      \
  ArrayXX operator OP(const A& a, const B& b) {                                             \
    return ArrayXX(internal::map2(a, b, [](double x, double y) { return x OP y; }));        \
  }                                                                                         \
  template <class A, std::enable_if_t<internal::is_arr_v<A>, int> = 0>                      \
  ArrayXX operator OP(const A& a, double s) {                                               \
    return ArrayXX(internal::map1(a, [s](double x) { return x OP s; }));                    \
  }                                                                                         \
  template <class A, std::enable_if_t<internal::is_arr_v<A>, int> = 0>                      \
  ArrayXX operator OP(double s, const A& a) {                                               \
    return ArrayXX(internal::map1(a, [s](double x) { return s OP x; }));                    \
  }
GBOPT_SUBSET_ARR_BINOP(+)
GBOPT_SUBSET_ARR_BINOP(-)
GBOPT_SUBSET_ARR_BINOP(*)
GBOPT_SUBSET_ARR_BINOP(/)
#undef GBOPT_SUBSET_ARR_BINOP
template <class A, std::enable_if_t<internal::is_arr_v<A>, int> = 0>
ArrayXX operator-(const A& a) { return ArrayXX(internal::map1(a, [](double x) { return -x; })); }

// Symmetric product from one stored triangle.
template <int UpLo, class B, std::enable_if_t<internal::is_mat_v<B>, int> = 0>
MatrixXd operator*(const SelfAdjointView<UpLo>& s, const B& b) {
  const internal::Dense& a = s.a;
  if (a.r_ != a.c_ || a.c_ != b.rows()) internal::fail("selfadjoint product shape");
  auto el = [&](Index i, Index j) {
    const bool lower = UpLo == Lower;
    return (lower ? (i >= j) : (i <= j)) ? a.at(i, j) : a.at(j, i);
  };
  MatrixXd c(a.r_, b.cols());
  for (Index j = 0; j < b.cols(); ++j)
    for (Index k = 0; k < a.c_; ++k) {
      const double bkj = b.at(k, j);
      for (Index i = 0; i < a.r_; ++i) c.at(i, j) += el(i, k) * bkj;
    }
  return c;
}

// ---------------------------------------------------------- permutations
template <int N = Dynamic>
class PermutationMatrix {
 public:
  struct Indices {
    std::vector<int> v;
    int& operator()(Index i) { return v[static_cast<size_t>(i)]; }
    int operator()(Index i) const { return v[static_cast<size_t>(i)]; }
    Index size() const { return static_cast<Index>(v.size()); }
  };
  struct Transposed {
    const PermutationMatrix* p;
  };
  explicit PermutationMatrix(Index n) { idx_.v.resize(static_cast<size_t>(n)); for (Index i = 0; i < n; ++i) idx_.v[static_cast<size_t>(i)] = static_cast<int>(i); }
  Indices& indices() { return idx_; }
  const Indices& indices() const { return idx_; }
  Transposed transpose() const { return Transposed{this}; }

 private:
  Indices idx_;
};
// (P A).row(indices(i)) = A.row(i)
template <int N, class A, std::enable_if_t<internal::is_mat_v<A>, int> = 0>
MatrixXd operator*(const PermutationMatrix<N>& p, const A& a) {
  MatrixXd out(a.rows(), a.cols());
  for (Index i = 0; i < a.rows(); ++i)
    for (Index j = 0; j < a.cols(); ++j) out(p.indices()(i), j) = a.at(i, j);
  return out;
}
// (A P^T).col(indices(j)) = A.col(j)
template <class A, std::enable_if_t<internal::is_mat_v<A>, int> = 0>
MatrixXd operator*(const A& a, const PermutationMatrix<Dynamic>::Transposed& pt) {
  MatrixXd out(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) out(i, pt.p->indices()(j)) = a.at(i, j);
  return out;
}

// --------------------------------------------------------- decompositions
// Householder QR (A = Q R, reflectors H_k = I - tau v v^T, v_0 = 1).
template <class M>
class HouseholderQR {
 public:
  explicit HouseholderQR(const MatrixXd& a) : qr_(a), tau_(std::min(a.rows(), a.cols())) {
    const Index m = qr_.rows(), n = qr_.cols();
    for (Index k = 0; k < std::min(m, n); ++k) {
      double sig = 0.0;
      for (Index i = k + 1; i < m; ++i) sig += qr_(i, k) * qr_(i, k);
      const double x0 = qr_(k, k);
      if (sig == 0.0) { tau_(k) = 0.0; continue; }
      const double nrm = std::sqrt(x0 * x0 + sig);
      const double beta = x0 >= 0.0 ? -nrm : nrm;
      const double v0 = x0 - beta;
      for (Index i = k + 1; i < m; ++i) qr_(i, k) /= v0;
      tau_(k) = (beta - x0) / beta;
      qr_(k, k) = beta;
      for (Index j = k + 1; j < n; ++j) {
        double s = qr_(k, j);
        for (Index i = k + 1; i < m; ++i) s += qr_(i, k) * qr_(i, j);
        s *= tau_(k);
        qr_(k, j) -= s;
        for (Index i = k + 1; i < m; ++i) qr_(i, j) -= s * qr_(i, k);
      }
    }
  }
  const MatrixXd& matrixQR() const { return qr_; }
  MatrixXd householderQ() const {
    const Index m = qr_.rows();
    MatrixXd q = MatrixXd::Identity(m, m);
    for (Index k = std::min(m, qr_.cols()) - 1; k >= 0; --k) {
      for (Index j = 0; j < m; ++j) {
        double s = q(k, j);
        for (Index i = k + 1; i < m; ++i) s += qr_(i, k) * q(i, j);
        s *= tau_(k);
        q(k, j) -= s;
        for (Index i = k + 1; i < m; ++i) q(i, j) -= s * qr_(i, k);
      }
    }
    return q;
  }

 private:
  MatrixXd qr_;
  VectorXd tau_;
};

// Eigenvalues of a symmetric matrix by cyclic Jacobi rotations, ascending.
template <class M>
class SelfAdjointEigenSolver {
 public:
  explicit SelfAdjointEigenSolver(const MatrixXd& a0) : ev_(a0.rows()) {
    MatrixXd a = a0;
    const Index n = a.rows();
    for (int sweep = 0; sweep < 100; ++sweep) {
      double off = 0.0, tot = 0.0;
      for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) {
          tot += a(i, j) * a(i, j);
          if (i != j) off += a(i, j) * a(i, j);
        }
      if (off <= 1e-32 * tot || off == 0.0) break;
      for (Index p = 0; p < n - 1; ++p)
        for (Index q = p + 1; q < n; ++q) {
          const double apq = a(p, q);
          if (apq == 0.0) continue;
          const double theta = (a(q, q) - a(p, p)) / (2.0 * apq);
          const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
          const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
          for (Index k = 0; k < n; ++k) {
            const double akp = a(k, p), akq = a(k, q);
            a(k, p) = c * akp - s * akq;
            a(k, q) = s * akp + c * akq;
          }
          for (Index k = 0; k < n; ++k) {
            const double apk = a(p, k), aqk = a(q, k);
            a(p, k) = c * apk - s * aqk;
            a(q, k) = s * apk + c * aqk;
          }
        }
    }
    std::vector<double> e(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) e[static_cast<size_t>(i)] = a(i, i);
    std::sort(e.begin(), e.end());
    for (Index i = 0; i < n; ++i) ev_(i) = e[static_cast<size_t>(i)];
  }
  const VectorXd& eigenvalues() const { return ev_; }

 private:
  VectorXd ev_;
};

}  // namespace Eigen
