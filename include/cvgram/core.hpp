#pragma once
// Core types of the B200 cvgram engine, source-compatible with the reference
// header /root/reference/proj/include/cvgram/core.hpp (same names, fields,
// exception types and messages).  Matrix / Vector / Index are the reference's
// own Eigen typedefs (core.hpp:16-18) whenever <Eigen/Dense> is on the include
// path, so callers that run Eigen operations on a FoldResult (.block, .ldlt,
// ...) compile unchanged; without Eigen (define CVGRAM_NO_EIGEN to force it)
// they are a small dense row-major fp64 type with the subset of Eigen the
// reference API and its tests use.  Computation happens in
// the sm_100a engine behind include/cvgram_b200.h; these headers only validate
// and marshal, touching matrices only through rows() / cols() / size() /
// data() / (i, j) / allFinite() / norm() -- the members both types share.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <initializer_list>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#if !defined(CVGRAM_NO_EIGEN) && defined(__has_include)
#if __has_include(<Eigen/Dense>)
#include <Eigen/Dense>
#define CVGRAM_WITH_EIGEN 1
#endif
#endif

namespace cvgram {

#ifdef CVGRAM_WITH_EIGEN
using Matrix = Eigen::Matrix<double, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor>;  // core.hpp:16
using Vector = Eigen::RowVectorXd;                                                       // core.hpp:17
using Index = Eigen::Index;                                                              // core.hpp:18
#else
using Index = std::ptrdiff_t;  // Eigen::Index (core.hpp:18)

class Matrix;

/// Dense row-major fp64 matrix (stands in for the reference's Eigen Matrix, core.hpp:16).
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols) : r_(rows), c_(cols), d_(static_cast<size_t>(rows * cols), 0.0) {}
  static Matrix Zero(Index rows, Index cols) { return Matrix(rows, cols); }
  static Matrix Constant(Index rows, Index cols, double v) {
    Matrix m(rows, cols);
    std::fill(m.d_.begin(), m.d_.end(), v);
    return m;
  }
  static Matrix Ones(Index rows, Index cols) { return Constant(rows, cols, 1.0); }
  static Matrix Identity(Index rows, Index cols) {
    Matrix m(rows, cols);
    for (Index i = 0; i < std::min(rows, cols); ++i) m(i, i) = 1.0;
    return m;
  }

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double& operator()(Index i, Index j) { return d_[static_cast<size_t>(i * c_ + j)]; }
  double operator()(Index i, Index j) const { return d_[static_cast<size_t>(i * c_ + j)]; }
  double& operator()(Index i) { return d_[static_cast<size_t>(i)]; }
  double operator()(Index i) const { return d_[static_cast<size_t>(i)]; }

  void setZero() { std::fill(d_.begin(), d_.end(), 0.0); }
  bool allFinite() const {
    for (double v : d_)
      if (!std::isfinite(v)) return false;
    return true;
  }
  bool isZero(double tol = 0.0) const {
    for (double v : d_)
      if (std::abs(v) > tol) return false;
    return true;
  }
  double maxAbs() const {
    double m = 0.0;
    for (double v : d_) m = std::max(m, std::abs(v));
    return m;
  }
  double norm() const {
    long double s = 0;
    for (double v : d_) s += static_cast<long double>(v) * v;
    return std::sqrt(static_cast<double>(s));
  }
  Matrix transpose() const {
    Matrix t(c_, r_);
    for (Index i = 0; i < r_; ++i)
      for (Index j = 0; j < c_; ++j) t(j, i) = (*this)(i, j);
    return t;
  }
  Matrix operator-(const Matrix& o) const { return zip(o, [](double a, double b) { return a - b; }); }
  Matrix operator+(const Matrix& o) const { return zip(o, [](double a, double b) { return a + b; }); }
  Matrix& operator-=(const Matrix& o) { return *this = *this - o; }
  Matrix& operator+=(const Matrix& o) { return *this = *this + o; }
  Matrix operator*(double s) const {
    Matrix m = *this;
    for (double& v : m.d_) v *= s;
    return m;
  }
  /// Plain host product for tests and small checks (not on the engine path).
  Matrix operator*(const Matrix& o) const {
    if (c_ != o.r_) throw std::invalid_argument("matrix product: shape mismatch");
    Matrix out(r_, o.c_);
    for (Index i = 0; i < r_; ++i)
      for (Index k = 0; k < c_; ++k) {
        const double a = (*this)(i, k);
        for (Index j = 0; j < o.c_; ++j) out(i, j) += a * o(k, j);
      }
    return out;
  }
  bool operator==(const Matrix& o) const { return r_ == o.r_ && c_ == o.c_ && d_ == o.d_; }
  bool operator!=(const Matrix& o) const { return !(*this == o); }

  /// Comma initializer: `m << 1, 2, 3;` fills row-major.
  class Filler {
   public:
    Filler(Matrix& m, double v) : m_(m), i_(0) { put(v); }
    Filler& operator,(double v) {
      put(v);
      return *this;
    }

   private:
    void put(double v) {
      if (i_ >= m_.size()) throw std::out_of_range("too many coefficients");
      m_.d_[static_cast<size_t>(i_++)] = v;
    }
    Matrix& m_;
    Index i_;
  };
  Filler operator<<(double v) { return Filler(*this, v); }

 private:
  template <typename F>
  Matrix zip(const Matrix& o, F f) const {
    if (r_ != o.r_ || c_ != o.c_) throw std::invalid_argument("elementwise op: shape mismatch");
    Matrix m(r_, c_);
    for (size_t i = 0; i < d_.size(); ++i) m.d_[i] = f(d_[i], o.d_[i]);
    return m;
  }
  Index r_ = 0, c_ = 0;
  std::vector<double> d_;
};

inline Matrix operator*(double s, const Matrix& m) { return m * s; }

/// Row vector (Eigen::RowVectorXd in the reference, core.hpp:17).
class Vector : public Matrix {
 public:
  Vector() = default;
  explicit Vector(Index n) : Matrix(1, n) {}
  Vector(const Matrix& m) : Matrix(m) {  // NOLINT: implicit like Eigen's
    if (m.rows() > 1 && m.cols() > 1) throw std::invalid_argument("not a vector");
  }
  static Vector Ones(Index n) {
    Vector v(n);
    for (Index i = 0; i < n; ++i) v(i) = 1.0;
    return v;
  }
  static Vector Zero(Index n) { return Vector(n); }
};

#endif  // CVGRAM_WITH_EIGEN

struct dimension_error : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

struct partition_error : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

/// Scaling requested but some training partition has fewer than two rows.
struct scalability_error : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

/// X (N x K) and Y (N x M), one sample per row; invariants of core.hpp:37-45.
class DatasetPair {
 public:
  DatasetPair(Matrix x, Matrix y) : x_(std::move(x)), y_(std::move(y)) {
    if (x_.rows() != y_.rows()) throw dimension_error("x and y must have the same number of rows");
    if (x_.rows() < 2) throw dimension_error("need at least 2 samples");
    if (x_.cols() < 1 || y_.cols() < 1) throw dimension_error("x and y must each have at least one column");
    if (!x_.allFinite() || !y_.allFinite()) throw dimension_error("x and y entries must be finite");
  }
  const Matrix& x() const { return x_; }
  const Matrix& y() const { return y_; }
  Index n_rows() const { return x_.rows(); }
  Index n_features() const { return x_.cols(); }
  Index n_responses() const { return y_.cols(); }

 private:
  Matrix x_;
  Matrix y_;
};

/// 1-based fold labels {1..p} (core.hpp:59-64).
struct Partitioning {
  std::vector<int> labels;
  int p = 0;
  Index n_rows() const { return static_cast<Index>(labels.size()); }
};

/// Four independent preprocessing flags (core.hpp:67-78).
struct PreprocessConfig {
  bool center_x = false;
  bool center_y = false;
  bool scale_x = false;
  bool scale_y = false;
  bool any_center() const { return center_x || center_y; }
  bool any_scale() const { return scale_x || scale_y; }
  bool any() const { return any_center() || any_scale(); }
  bool operator==(const PreprocessConfig&) const = default;
  /// enumerate_configs bit order (combos.hpp:33-45)
  uint32_t mask() const {
    return (center_x ? 8u : 0u) | (center_y ? 4u : 0u) | (scale_x ? 2u : 0u) | (scale_y ? 1u : 0u);
  }
};

struct DeviceGlobal;  // engine.hpp: device state behind a GlobalCache

/// Whole-dataset aggregates (core.hpp:83-93).  `device` keeps the engine's
/// shifted-basis products so fold_products never recomputes them.
struct GlobalCache {
  Matrix xtx;
  Matrix xty;
  Vector mean_x;
  Vector mean_y;
  Vector sum_x;
  Vector sum_y;
  Vector sum_sq_x;
  Vector sum_sq_y;
  Index n_rows = 0;
  std::shared_ptr<DeviceGlobal> device;
};

struct FoldStats {
  Vector mean_x_t;
  Vector mean_y_t;
  Vector std_x_t;
  Vector std_y_t;
  Index n_train = 0;
  Index n_val = 0;
};

struct FoldResult {
  int fold_id = 0;
  Matrix xtx_t;
  Matrix xty_t;
  FoldStats stats;
};

/// Largest entrywise |a-b| / max(|a|, |b|, floor) (core.hpp:133-150).
inline double max_rel_diff(const Matrix& a, const Matrix& b, double floor = 1e-30) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) throw dimension_error("max_rel_diff: shape mismatch");
  double worst = 0.0;
  const double* pa = a.data();
  const double* pb = b.data();
  for (Index i = 0; i < a.size(); ++i) {
    const double den = std::max({std::abs(pa[i]), std::abs(pb[i]), floor});
    worst = std::max(worst, std::abs(pa[i] - pb[i]) / den);
  }
  return worst;
}

/// ||a-b||_F / max(||a||_F, ||b||_F, floor) (core.hpp:153-156).
inline double rel_frobenius_dist(const Matrix& a, const Matrix& b, double floor = 1e-30) {
  return (a - b).norm() / std::max({a.norm(), b.norm(), floor});
}

}  // namespace cvgram

// hadamard_outer_divide (core.hpp:116-130) runs on the device: engine.hpp.
#include "cvgram/engine.hpp"
