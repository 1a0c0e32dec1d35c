// isnmf-b200 C++ API — dense column-major fp64 carriers.
//
// The reference uses Eigen::MatrixXd / VectorXd (proj/include/isnmf/matrix.hpp:14-16);
// Eigen is not part of this build, so Matrix / Vector are small owning
// column-major types with the members the API and its callers use (rows, cols,
// size, data, (i, j), col, Zero / Ones / Constant, sum / mean / norm /
// allFinite) plus products for test convenience.  Layout and meaning match
// Eigen's defaults, so data() pointers can be exchanged with Eigen users.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <initializer_list>
#include <string>
#include <vector>

#include "errors.hpp"

namespace isnmf {

using Index = std::ptrdiff_t;

class Vector {
 public:
  Vector() = default;
  explicit Vector(Index n) : d_(static_cast<size_t>(n), 0.0) {}
  Vector(std::initializer_list<double> v) : d_(v) {}
  static Vector Zero(Index n) { return Vector(n); }
  static Vector Ones(Index n) { return Constant(n, 1.0); }
  static Vector Constant(Index n, double v) {
    Vector x(n);
    std::fill(x.d_.begin(), x.d_.end(), v);
    return x;
  }
  Index size() const { return static_cast<Index>(d_.size()); }
  void resize(Index n) { d_.resize(static_cast<size_t>(n)); }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double& operator[](Index i) { return d_[static_cast<size_t>(i)]; }
  double operator[](Index i) const { return d_[static_cast<size_t>(i)]; }
  double& operator()(Index i) { return (*this)[i]; }
  double operator()(Index i) const { return (*this)[i]; }
  double sum() const {
    double s = 0.0;
    for (double x : d_) s += x;
    return s;
  }
  double mean() const { return sum() / static_cast<double>(d_.size()); }
  bool allFinite() const {
    for (double x : d_)
      if (!std::isfinite(x)) return false;
    return true;
  }
  double maxAbs() const {
    double m = 0.0;
    for (double x : d_) m = std::max(m, std::abs(x));
    return m;
  }

 private:
  std::vector<double> d_;
};

class Matrix {
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols) : r_(rows), c_(cols), d_(static_cast<size_t>(rows * cols), 0.0) {}
  static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
  static Matrix Ones(Index r, Index c) { return Constant(r, c, 1.0); }
  static Matrix Constant(Index r, Index c, double v) {
    Matrix m(r, c);
    std::fill(m.d_.begin(), m.d_.end(), v);
    return m;
  }
  /// A one-column matrix holding v (Eigen's implicit vector -> matrix).
  static Matrix FromVector(const Vector& v) {
    Matrix m(v.size(), 1);
    std::copy(v.data(), v.data() + v.size(), m.data());
    return m;
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double& operator()(Index i, Index j) { return d_[static_cast<size_t>(j * r_ + i)]; }
  double operator()(Index i, Index j) const { return d_[static_cast<size_t>(j * r_ + i)]; }
  double* col_data(Index j) { return d_.data() + j * r_; }
  const double* col_data(Index j) const { return d_.data() + j * r_; }
  Vector col(Index j) const {
    Vector v(r_);
    std::copy(col_data(j), col_data(j) + r_, v.data());
    return v;
  }
  void set_col(Index j, const Vector& v) { std::copy(v.data(), v.data() + r_, col_data(j)); }
  void setZero() { std::fill(d_.begin(), d_.end(), 0.0); }
  double sum() const {
    double s = 0.0;
    for (double x : d_) s += x;
    return s;
  }
  double mean() const { return sum() / static_cast<double>(d_.size()); }
  double norm() const {
    double s = 0.0;
    for (double x : d_) s += x * x;
    return std::sqrt(s);
  }
  double maxAbs() const {
    double m = 0.0;
    for (double x : d_) m = std::max(m, std::abs(x));
    return m;
  }
  bool allFinite() const {
    for (double x : d_)
      if (!std::isfinite(x)) return false;
    return true;
  }
  bool anyNegative() const {
    for (double x : d_)
      if (x < 0.0) return true;
    return false;
  }
  Matrix operator-(const Matrix& o) const {
    Matrix m(r_, c_);
    for (size_t i = 0; i < d_.size(); ++i) m.d_[i] = d_[i] - o.d_[i];
    return m;
  }
  Matrix operator+(const Matrix& o) const {
    Matrix m(r_, c_);
    for (size_t i = 0; i < d_.size(); ++i) m.d_[i] = d_[i] + o.d_[i];
    return m;
  }
  Matrix operator*(double s) const {
    Matrix m(r_, c_);
    for (size_t i = 0; i < d_.size(); ++i) m.d_[i] = d_[i] * s;
    return m;
  }
  /// Host product (test convenience; the engine's products run on the device).
  Matrix operator*(const Matrix& o) const {
    Matrix m(r_, o.c_);
    for (Index j = 0; j < o.c_; ++j)
      for (Index k = 0; k < c_; ++k) {
        const double b = o(k, j);
        for (Index i = 0; i < r_; ++i) m(i, j) += (*this)(i, k) * b;
      }
    return m;
  }
  Vector operator*(const Vector& v) const {
    Vector y(r_);
    for (Index k = 0; k < c_; ++k)
      for (Index i = 0; i < r_; ++i) y[i] += (*this)(i, k) * v[k];
    return y;
  }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> d_;
};

inline Matrix operator*(double s, const Matrix& m) { return m * s; }

// matrix.hpp:18-29
inline void require_same_shape(const Matrix& a, const Matrix& b, const char* what) {
  if (a.rows() != b.rows() || a.cols() != b.cols())
    throw ShapeMismatch(std::string(what) + ": " + std::to_string(a.rows()) + "x" + std::to_string(a.cols()) +
                        " vs " + std::to_string(b.rows()) + "x" + std::to_string(b.cols()));
}

inline void require_same_size(const Vector& a, const Vector& b, const char* what) {
  if (a.size() != b.size())
    throw ShapeMismatch(std::string(what) + ": " + std::to_string(a.size()) + " vs " + std::to_string(b.size()));
}

// matrix.hpp:32-35
inline void require_nonneg_finite(const Matrix& m, const char* what) {
  if (!m.allFinite()) throw NonFiniteEntry(std::string(what) + ": non-finite entry");
  if (m.anyNegative()) throw NegativeEntry(std::string(what) + ": negative entry");
}

/// || a - b ||_F, the stopping statistic of the trainers (matrix.hpp:38-41).
inline double frobenius_delta(const Matrix& w_new, const Matrix& w_old) {
  require_same_shape(w_new, w_old, "frobenius_delta");
  return (w_new - w_old).norm();
}

}  // namespace isnmf
