// isnmf-b200 C++ API — the numerical kernels of the reference
// (proj/include/isnmf/kernels.hpp:30-183) on the B200 engine.  Shapes and
// arguments are checked here with the reference's exception types; the
// arithmetic runs on the device in fp32 (fp64 accumulation of sums) through
// the C ABI.  aux_value / aux_constant are diagnostics (majorisation tests) and
// are evaluated on the host in fp64.
#pragma once

#include <cmath>

#include "errors.hpp"
#include "matrix.hpp"

namespace isnmf {

namespace detail {
inline void require_epsilon(double epsilon) {
  if (!(epsilon > 0.0)) throw NegativeInput("epsilon must be > 0");
}
inline void require_vwh(const Matrix& v, const Matrix& w, const Matrix& h, const char* what) {
  if (w.rows() != v.rows() || w.cols() != h.rows() || h.cols() != v.cols())
    throw ShapeMismatch(std::string(what) + ": inconsistent shapes");
}
}  // namespace detail

/// sum_i is_term((y_i - x_i)/(eps + x_i))  (kernels.hpp:30-40).
inline double is_divergence(const Vector& y, const Vector& x, double epsilon) {
  require_same_size(y, x, "is_divergence");
  double out = 0.0;
  detail::check(isnmf_is_divergence(y.data(), y.size(), x.data(), x.size(), epsilon, &out));
  return out;
}

/// (1/N) sum_n d_IS(eps + v_n, eps + W h_n)  (kernels.hpp:43-55).
inline double objective(const Matrix& v, const Matrix& w, const Matrix& h, double epsilon) {
  detail::require_epsilon(epsilon);
  detail::require_vwh(v, w, h, "objective");
  if (v.cols() == 0) throw EmptyDataset("objective: no columns");
  double out = 0.0;
  detail::check(isnmf_objective(v.data(), w.data(), h.data(), w.rows(), w.cols(), v.cols(), epsilon, &out));
  return out;
}

/// `iters` MM updates of h at fixed W  (kernels.hpp:62-80).
inline Vector solve_h(const Vector& v, const Matrix& w, const Vector& h0, int iters, double epsilon) {
  detail::require_epsilon(epsilon);
  if (v.size() != w.rows()) throw ShapeMismatch("solve_h: v vs W rows");
  if (h0.size() != w.cols()) throw ShapeMismatch("solve_h: h0 vs W cols");
  Vector h(h0.size());
  detail::check(isnmf_solve_h(v.data(), w.data(), h0.data(), w.rows(), w.cols(), 1, iters, epsilon, h.data()));
  return h;
}

/// Batched solve_h: every column of v from the matching column of h0.
inline Matrix solve_h(const Matrix& v, const Matrix& w, const Matrix& h0, int iters, double epsilon) {
  detail::require_epsilon(epsilon);
  detail::require_vwh(v, w, h0, "solve_h");
  Matrix h(h0.rows(), h0.cols());
  detail::check(isnmf_solve_h(v.data(), w.data(), h0.data(), w.rows(), w.cols(), v.cols(), iters, epsilon,
                              h.data()));
  return h;
}

/// a_fk = (e+v_f)/(e+(Wh)_f)^2 h_k W_fk^2,  b_fk = h_k/(e+(Wh)_f)  (kernels.hpp:86-89).
struct SampleStats {
  Matrix a;
  Matrix b;
};

/// Full-data statistics, the sum of sample_stats over the columns (kernels.hpp:125-137).
inline SampleStats batch_stats(const Matrix& v, const Matrix& w, const Matrix& h, double epsilon) {
  detail::require_epsilon(epsilon);
  detail::require_vwh(v, w, h, "batch_stats");
  SampleStats s{Matrix(w.rows(), w.cols()), Matrix(w.rows(), w.cols())};
  detail::check(isnmf_batch_stats(v.data(), w.data(), h.data(), w.rows(), w.cols(), v.cols(), epsilon, s.a.data(),
                                  s.b.data()));
  return s;
}

/// Per-sample statistics  (kernels.hpp:112-121).
inline SampleStats sample_stats(const Vector& v, const Matrix& w, const Vector& h, double epsilon) {
  detail::require_epsilon(epsilon);
  if (v.size() != w.rows() || h.size() != w.cols()) throw ShapeMismatch("sample_stats: inconsistent shapes");
  return batch_stats(Matrix::FromVector(v), w, Matrix::FromVector(h), epsilon);
}

/// W = sqrt(A/B); A = B = 0 keeps the previous entry  (kernels.hpp:142-159).
inline Matrix update_w(const Matrix& a, const Matrix& b, const Matrix& w_prev) {
  require_same_shape(a, b, "update_w: a vs b");
  require_same_shape(a, w_prev, "update_w: a vs w_prev");
  Matrix w(a.rows(), a.cols());
  detail::check(isnmf_update_w(a.data(), b.data(), w_prev.data(), a.rows(), a.cols(), w.data()));
  return w;
}

/// sum_fk a_fk/W_fk + b_fk W_fk  (kernels.hpp:163-167; host diagnostic).
inline double aux_value(const Matrix& a, const Matrix& b, const Matrix& w) {
  require_same_shape(a, b, "aux_value: a vs b");
  require_same_shape(a, w, "aux_value: a vs w");
  double s = 0.0;
  for (Index i = 0; i < a.size(); ++i) s += a.data()[i] / w.data()[i] + b.data()[i] * w.data()[i];
  return s;
}

/// Constant completing the auxiliary function at w_anchor (kernels.hpp:173-183; host diagnostic).
inline double aux_constant(const Matrix& v, const Matrix& w_anchor, const Matrix& h, double epsilon) {
  detail::require_epsilon(epsilon);
  detail::require_vwh(v, w_anchor, h, "aux_constant");
  const Matrix x = w_anchor * h;
  double s = 0.0;
  for (Index i = 0; i < v.size(); ++i) {
    const double ve = v.data()[i] + epsilon, xh = x.data()[i] + epsilon;
    s += epsilon * ve / (xh * xh) + epsilon / xh - std::log(ve / xh) - 2.0;
  }
  return s;
}

}  // namespace isnmf
