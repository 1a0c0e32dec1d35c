// TEST INFRASTRUCTURE ONLY — the CPU fp64 oracle for the isnmf-b200 engine.
//
// A from-scratch restatement (no Eigen, plain loops) of the arithmetic of the
// reference's online / batch Itakura-Saito NMF path in
// /root/reference/proj/include/isnmf/{kernels,model,matrix,rng,online,batch}.hpp.
// Every function cites the reference lines it follows.  Only tests/, the
// __graft_entry__.smoke() checker and bench.py's cpu_baseline / --impl reference
// leg may use it; the product (paper_1106_4198_b200/, include/) never does.
//
// Parity status:
//  * pinned    — is_divergence, objective, solve_h, sample_stats, batch_stats,
//                update_w, aux_value/aux_constant, rescale_dictionary,
//                frobenius_delta, config defaults: checked against every golden
//                value and property of proj/tests/test_core.cpp and
//                proj/tests/test_kernels.cpp (tests/test_oracle_golden.py).
//  * unpinned  — online_step / dictionary_commit / online_resume / batch_train:
//                the reference ships no test for them (tests/CMakeLists.txt:7-10
//                lists test_online.cpp / test_batch.cpp, absent) and the
//                reference cannot be compiled here (Eigen3 absent).  They are
//                held to the SPEC.md examples and acceptance properties instead
//                (tests/test_oracle_trainers.py), "parity unpinned" beyond that.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace isnmf_oracle {

// ---- errors (reference errors.hpp:9-90), carried as a code -----------------
enum Code : int {
  OK = 0,
  SHAPE_MISMATCH = 1,
  EMPTY_DATASET = 2,
  NEGATIVE_INPUT = 3,
  NON_POSITIVE_INIT = 4,
  ZERO_COLUMN = 5,
  INCONSISTENT_STATS = 6,
  NUMERICAL_FAILURE = 7,
  DIVERGED_OBJECTIVE = 8,
  NON_FINITE_ENTRY = 9,
  NEGATIVE_ENTRY = 10,
  IO_ERROR = 11,
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// ---- column-major fp64 matrix (reference matrix.hpp:14-16 uses Eigen) ------
struct Mat {
  int64_t r = 0, c = 0;
  std::vector<double> d;
  Mat() = default;
  Mat(int64_t rows, int64_t cols, double fill = 0.0) : r(rows), c(cols), d(size_t(rows * cols), fill) {}
  double& operator()(int64_t i, int64_t j) { return d[size_t(j * r + i)]; }
  double operator()(int64_t i, int64_t j) const { return d[size_t(j * r + i)]; }
  double* col(int64_t j) { return d.data() + j * r; }
  const double* col(int64_t j) const { return d.data() + j * r; }
  int64_t size() const { return r * c; }
};

inline bool all_finite(const Mat& m) {
  for (double x : m.d)
    if (!std::isfinite(x)) return false;
  return true;
}

// ---- rng (reference rng.hpp:10-44) ------------------------------------------
inline uint64_t splitmix64(uint64_t x) {  // rng.hpp:10-15
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
inline uint64_t mix_seed(uint64_t seed, uint64_t stream) {  // rng.hpp:17-19
  return splitmix64(splitmix64(seed) ^ splitmix64(~stream));
}
inline std::mt19937_64 make_engine(uint64_t seed) {  // rng.hpp:21-23
  return std::mt19937_64(splitmix64(seed));
}
inline double uniform01(std::mt19937_64& g) {  // rng.hpp:27-29
  return static_cast<double>(g() >> 11) * 0x1.0p-53;
}
inline double uniform_open01(std::mt19937_64& g) { return 1.0 - uniform01(g); }  // rng.hpp:32-34
inline uint64_t uniform_below(std::mt19937_64& g, uint64_t n) {  // rng.hpp:37-44
  const uint64_t limit = ~uint64_t(0) - (~uint64_t(0) % n);
  uint64_t x;
  do {
    x = g();
  } while (x >= limit);
  return x % n;
}

// ---- kernels (reference kernels.hpp) ----------------------------------------
inline double is_term(double u) {  // kernels.hpp:15-18
  const double t = u - std::log1p(u);
  return t > 0.0 ? t : 0.0;
}
inline void require_epsilon(double eps) {  // kernels.hpp:20-22
  if (!(eps > 0.0)) throw Error(NEGATIVE_INPUT, "epsilon must be > 0");
}

// kernels.hpp:30-40
inline double is_divergence(const double* y, const double* x, int64_t n, int64_t nx, double eps) {
  if (n != nx) throw Error(SHAPE_MISMATCH, "is_divergence: size mismatch");
  require_epsilon(eps);
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (y[i] < 0.0 || x[i] < 0.0) throw Error(NEGATIVE_INPUT, "is_divergence: negative entry");
    acc += is_term((y[i] - x[i]) / (eps + x[i]));
  }
  return acc;
}

// Inner product; the simd reduction lets the compiler reassociate like Eigen's
// vectorised transposed GEMV does (kernels.hpp:74,76).
inline double dot(const double* a, const double* b, int64_t n) {
  double s = 0.0;
#pragma omp simd reduction(+ : s)
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

// y = W h (no epsilon), plain column sweep.
inline void gemv(const Mat& w, const double* h, double* y) {
  for (int64_t f = 0; f < w.r; ++f) y[f] = 0.0;
  for (int64_t k = 0; k < w.c; ++k) {
    const double hk = h[k];
    const double* wk = w.col(k);
    for (int64_t f = 0; f < w.r; ++f) y[f] += wk[f] * hk;
  }
}

// kernels.hpp:43-55 — mean over frames of d_IS(e+v_n, e+W h_n)
inline double objective(const Mat& v, const Mat& w, const Mat& h, double eps) {
  require_epsilon(eps);
  if (w.r != v.r || w.c != h.r || h.c != v.c) throw Error(SHAPE_MISMATCH, "objective: inconsistent V/W/H shapes");
  if (v.c == 0) throw Error(EMPTY_DATASET, "objective: no columns");
  std::vector<double> a(static_cast<size_t>(v.r));
  double acc = 0.0;
  for (int64_t n = 0; n < v.c; ++n) {
    gemv(w, h.col(n), a.data());
    const double* pv = v.col(n);
    for (int64_t f = 0; f < v.r; ++f) acc += is_term((pv[f] - a[f]) / (eps + a[f]));
  }
  return acc / static_cast<double>(v.c);
}

// kernels.hpp:62-80 — MM iterations for one frame; h updated in place.
inline void solve_h(const double* v, const Mat& w, double* h, int iters, double eps,
                    std::vector<double>& approx, std::vector<double>& ratio) {
  const int64_t F = w.r, K = w.c;
  approx.resize(size_t(F));
  ratio.resize(size_t(F));
  std::vector<double> num(static_cast<size_t>(K)), den(static_cast<size_t>(K));
  for (int it = 0; it < iters; ++it) {
    gemv(w, h, approx.data());
    for (int64_t f = 0; f < F; ++f) approx[f] += eps;
    for (int64_t f = 0; f < F; ++f) ratio[f] = (v[f] + eps) / (approx[f] * approx[f]);
    for (int64_t k = 0; k < K; ++k) num[size_t(k)] = dot(w.col(k), ratio.data(), F);
    for (int64_t f = 0; f < F; ++f) ratio[f] = 1.0 / approx[f];
    for (int64_t k = 0; k < K; ++k) den[size_t(k)] = dot(w.col(k), ratio.data(), F);
    for (int64_t k = 0; k < K; ++k) h[k] *= std::sqrt(num[size_t(k)] / den[size_t(k)]);
  }
}

inline void solve_h_checked(const double* v, int64_t nv, const Mat& w, const double* h0, int64_t nh, int iters,
                            double eps, double* h_out) {
  require_epsilon(eps);
  if (nv != w.r) throw Error(SHAPE_MISMATCH, "solve_h: v vs W rows");
  if (nh != w.c) throw Error(SHAPE_MISMATCH, "solve_h: h0 vs W cols");
  for (int64_t k = 0; k < nh; ++k)
    if (h0[k] <= 0.0) throw Error(NON_POSITIVE_INIT, "solve_h: h0 must be positive");
  std::copy(h0, h0 + nh, h_out);
  std::vector<double> a, r;
  solve_h(v, w, h_out, iters, eps, a, r);
}

// kernels.hpp:95-108 — adds one frame's statistics; approx := eps + W h.
inline void accumulate_sample_stats(const double* v, const Mat& w, const double* h, double eps, Mat& a_acc,
                                    Mat& b_acc, std::vector<double>& approx) {
  const int64_t F = w.r;
  approx.resize(size_t(F));
  gemv(w, h, approx.data());
  for (int64_t f = 0; f < F; ++f) approx[f] += eps;
  for (int64_t k = 0; k < w.c; ++k) {
    const double hk = h[k];
    if (hk == 0.0) continue;
    const double* wk = w.col(k);
    double* ak = a_acc.col(k);
    double* bk = b_acc.col(k);
    for (int64_t f = 0; f < F; ++f) {
      ak[f] += hk * (wk[f] * wk[f]) * (v[f] + eps) / (approx[f] * approx[f]);
      bk[f] += hk / approx[f];
    }
  }
}

// kernels.hpp:125-137 — full-data statistics (O(FKN)).
inline void batch_stats(const Mat& v, const Mat& w, const Mat& h, double eps, Mat& a, Mat& b) {
  require_epsilon(eps);
  if (w.r != v.r || w.c != h.r || h.c != v.c) throw Error(SHAPE_MISMATCH, "batch_stats: inconsistent shapes");
  const int64_t F = w.r, K = w.c;
  a = Mat(F, K);
  b = Mat(F, K);
  std::vector<double> ap(static_cast<size_t>(F));
  for (int64_t n = 0; n < v.c; ++n) {
    gemv(w, h.col(n), ap.data());
    const double* pv = v.col(n);
    const double* hn = h.col(n);
    for (int64_t k = 0; k < K; ++k) {
      double* ak = a.col(k);
      double* bk = b.col(k);
      for (int64_t f = 0; f < F; ++f) {
        const double x = ap[f] + eps;
        ak[f] += (pv[f] + eps) / (x * x) * hn[k];
        bk[f] += hn[k] / x;
      }
    }
  }
  for (int64_t i = 0; i < a.size(); ++i) a.d[size_t(i)] *= w.d[size_t(i)] * w.d[size_t(i)];
}

// kernels.hpp:142-159 — W = sqrt(A/B); dead entries keep w_prev.
inline Mat update_w(const Mat& a, const Mat& b, const Mat& w_prev) {
  if (a.r != b.r || a.c != b.c) throw Error(SHAPE_MISMATCH, "update_w: a vs b");
  if (a.r != w_prev.r || a.c != w_prev.c) throw Error(SHAPE_MISMATCH, "update_w: a vs w_prev");
  Mat w(a.r, a.c);
  for (int64_t i = 0; i < a.size(); ++i) {
    const double ai = a.d[size_t(i)], bi = b.d[size_t(i)];
    if (bi > 0.0)
      w.d[size_t(i)] = std::sqrt(ai / bi);
    else if (ai > 0.0)
      throw Error(INCONSISTENT_STATS, "update_w: a > 0 with b = 0");
    else
      w.d[size_t(i)] = w_prev.d[size_t(i)];
  }
  return w;
}

// kernels.hpp:163-167
inline double aux_value(const Mat& a, const Mat& b, const Mat& w) {
  if (a.r != b.r || a.c != b.c || a.r != w.r || a.c != w.c) throw Error(SHAPE_MISMATCH, "aux_value: shapes");
  double s = 0.0;
  for (int64_t i = 0; i < a.size(); ++i) s += a.d[size_t(i)] / w.d[size_t(i)] + b.d[size_t(i)] * w.d[size_t(i)];
  return s;
}

// kernels.hpp:173-183
inline double aux_constant(const Mat& v, const Mat& w, const Mat& h, double eps) {
  require_epsilon(eps);
  if (w.r != v.r || w.c != h.r || h.c != v.c) throw Error(SHAPE_MISMATCH, "aux_constant: inconsistent shapes");
  std::vector<double> ap(static_cast<size_t>(v.r));
  double s = 0.0;
  for (int64_t n = 0; n < v.c; ++n) {
    gemv(w, h.col(n), ap.data());
    for (int64_t f = 0; f < v.r; ++f) {
      const double ve = v(f, n) + eps, xh = ap[f] + eps;
      s += eps * ve / (xh * xh) + eps / xh - std::log(ve / xh) - 2.0;
    }
  }
  return s;
}

// matrix.hpp:38-41
inline double frobenius_delta(const Mat& a, const Mat& b) {
  if (a.r != b.r || a.c != b.c) throw Error(SHAPE_MISMATCH, "frobenius_delta");
  double s = 0.0;
  for (int64_t i = 0; i < a.size(); ++i) {
    const double d = a.d[size_t(i)] - b.d[size_t(i)];
    s += d * d;
  }
  return std::sqrt(s);
}

// ---- model (reference model.hpp) --------------------------------------------
enum class Restart { warm = 0, fresh = 1 };

struct Config {  // model.hpp:33-68
  int k = 8;
  double epsilon = 1e-12;
  double eta = -1.0;
  int beta = 1000;
  double r = 0.7;
  int inner_iters = 0;
  Restart restart = Restart::warm;
  uint64_t seed = 1;
  int n_seeds = 5;
  uint64_t max_epochs_or_samples = 500;
  double init_stats_weight = 1.0;

  void validate() const {  // model.hpp:48-57
    if (k < 1) throw Error(NEGATIVE_INPUT, "config: k must be >= 1");
    if (!(epsilon > 0.0)) throw Error(NEGATIVE_INPUT, "config: epsilon must be > 0");
    if (beta < 1) throw Error(NEGATIVE_INPUT, "config: beta must be >= 1");
    if (!(r >= 0.0 && r <= 1.0)) throw Error(NEGATIVE_INPUT, "config: r must be in [0,1]");
    if (inner_iters < 0) throw Error(NEGATIVE_INPUT, "config: inner_iters must be >= 0");
    if (n_seeds < 1) throw Error(NEGATIVE_INPUT, "config: n_seeds must be >= 1");
    if (!(init_stats_weight >= 0.0)) throw Error(NEGATIVE_INPUT, "config: init_stats_weight must be >= 0");
  }
  int effective_inner_iters() const {  // model.hpp:59-62
    if (inner_iters > 0) return inner_iters;
    return restart == Restart::warm ? 1 : 100;
  }
  double effective_eta(int64_t f, int64_t k_) const {  // model.hpp:64-67
    if (eta >= 0.0) return eta;
    return 1e-6 * std::sqrt(static_cast<double>(f) * static_cast<double>(k_));
  }
};

// model.hpp:73-86 — l1 column renormalisation with A/B/(H) compensation.
inline void rescale_dictionary(Mat& w, Mat& a, Mat& b, Mat* warm_h) {
  if (w.r != a.r || w.c != a.c) throw Error(SHAPE_MISMATCH, "rescale_dictionary: w vs a");
  if (w.r != b.r || w.c != b.c) throw Error(SHAPE_MISMATCH, "rescale_dictionary: w vs b");
  if (warm_h && warm_h->r != w.c) throw Error(SHAPE_MISMATCH, "rescale_dictionary: warm_h rows vs W cols");
  for (int64_t k = 0; k < w.c; ++k) {
    double s = 0.0;
    for (int64_t f = 0; f < w.r; ++f) s += w(f, k);
    if (!(s > 0.0)) throw Error(ZERO_COLUMN, "rescale_dictionary: dead atom " + std::to_string(k));
    for (int64_t f = 0; f < w.r; ++f) {
      w(f, k) /= s;
      a(f, k) /= s;
      b(f, k) *= s;
    }
    if (warm_h)
      for (int64_t n = 0; n < warm_h->c; ++n) (*warm_h)(k, n) *= s;
  }
}

// batch.hpp:58-70
inline Mat init_from_samples(const Mat& v, int k, uint64_t seed, double eps) {
  if (v.c < 1) throw Error(EMPTY_DATASET, "init_from_samples: empty dataset");
  if (k < 1) throw Error(NEGATIVE_INPUT, "init_from_samples: k must be >= 1");
  auto rng = make_engine(mix_seed(seed, 0x57696e6974ULL));
  Mat w(v.r, k);
  for (int j = 0; j < k; ++j) {
    const auto idx = int64_t(uniform_below(rng, uint64_t(v.c)));
    double s = 0.0;
    for (int64_t f = 0; f < v.r; ++f) {
      w(f, j) = std::max(v(f, idx), eps);
      s += w(f, j);
    }
    for (int64_t f = 0; f < v.r; ++f) w(f, j) /= s;
  }
  return w;
}

inline double mean(const double* p, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += p[i];
  return s / double(n);
}

// batch.hpp:74-78
inline Mat default_h0(const Mat& v, const Mat& w, double eps) {
  const double scale = std::max(mean(v.d.data(), v.size()), eps) / (double(w.c) * mean(w.d.data(), w.size()));
  return Mat(w.c, v.c, scale);
}

// harness.hpp:17-37 — held-out fit: H from one seed-deterministic stream of
// open-interval uniforms (column-major fill) scaled by max(mean V, eps)/(K mean W),
// `iters` MM updates at frozen W, then the mean divergence per frame.
inline Mat heldout_h0(const Mat& w, const Mat& test, double eps, uint64_t seed) {
  const double scale = std::max(mean(test.d.data(), test.size()), eps) / (double(w.c) * mean(w.d.data(), w.size()));
  std::mt19937_64 g = make_engine(mix_seed(seed, 0xE7A1ULL));
  Mat h(w.c, test.c);
  for (int64_t j = 0; j < h.c; ++j)
    for (int64_t i = 0; i < h.r; ++i) h(i, j) = scale * uniform_open01(g);
  return h;
}

inline double evaluate_heldout(const Mat& w, const Mat& test, double eps, int iters, uint64_t seed) {
  if (w.r != test.r) throw Error(SHAPE_MISMATCH, "evaluate_heldout: W rows vs test rows");
  if (test.c == 0) throw Error(EMPTY_DATASET, "evaluate_heldout: empty test set");
  Mat h = heldout_h0(w, test, eps, seed);
  std::vector<double> approx, ratio;
  for (int64_t j = 0; j < test.c; ++j) solve_h(test.col(j), w, h.col(j), iters, eps, approx, ratio);
  return objective(test, w, h, eps);
}

// ---- sample orders (reference online.hpp:53-149) ------------------------------
// CyclingSource::load_cycle (online.hpp:79-87): Fisher-Yates of [0,n).
inline std::vector<uint64_t> cycle_permutation(uint64_t seed, uint64_t cycle, uint64_t n) {
  std::vector<uint64_t> p(static_cast<size_t>(n));
  std::iota(p.begin(), p.end(), uint64_t(0));
  auto rng = make_engine(mix_seed(seed, cycle));
  for (size_t i = p.size(); i > 1; --i) std::swap(p[i - 1], p[size_t(uniform_below(rng, i))]);
  return p;
}

// ---- online trainer (reference online.hpp:224-419) ----------------------------
struct TracePoint {
  uint64_t samples;
  double train_obj;
};

struct Online {
  Mat w, a, b, pending_a, pending_b, warm_h;
  uint64_t t = 0;
  double rho = 1.0;
  Restart restart = Restart::fresh;
  uint64_t seed = 0;
  double last_delta = std::numeric_limits<double>::infinity();
  uint64_t commits = 0;
  double pending_div = 0.0;
  uint64_t pending_count = 0;
  double last_minibatch_obj = 0.0;
  std::vector<TracePoint> trace;
  double final_train_obj = 0.0;
  std::vector<double> scratch_approx, scratch_ratio, scratch_h;
};

// online.hpp:254-288 (dataset given as F x N when warm).
inline Online make_online_state(const Mat& w0, const Config& cfg, bool sized, uint64_t dataset_size,
                                const Mat* dataset) {
  cfg.validate();
  for (double x : w0.d)
    if (x < 0.0 || !std::isfinite(x)) throw Error(NON_POSITIVE_INIT, "online: W0 must be nonnegative and finite");
  for (int64_t k = 0; k < w0.c; ++k) {
    double s = 0.0;
    for (int64_t f = 0; f < w0.r; ++f) s += w0(f, k);
    if (!(s > 0.0)) throw Error(ZERO_COLUMN, "online: W0 has an all-zero column");
    if (std::abs(s - 1.0) > 1e-8) throw Error(NON_POSITIVE_INIT, "online: W0 columns must be l1-normalized");
  }
  Online st;
  st.w = w0;
  st.a = Mat(w0.r, w0.c);
  for (int64_t i = 0; i < w0.size(); ++i) st.a.d[size_t(i)] = cfg.init_stats_weight * w0.d[size_t(i)] * w0.d[size_t(i)];
  st.b = Mat(w0.r, w0.c, cfg.init_stats_weight);
  st.pending_a = Mat(w0.r, w0.c);
  st.pending_b = Mat(w0.r, w0.c);
  st.restart = cfg.restart;
  st.seed = cfg.seed;
  st.rho = sized ? std::pow(cfg.r, double(cfg.beta) / double(dataset_size)) : 1.0;
  if (cfg.restart == Restart::warm) {
    if (!dataset) throw Error(EMPTY_DATASET, "online: warm restarts need an in-memory dataset");
    st.warm_h = default_h0(*dataset, w0, cfg.epsilon);
  }
  return st;
}

// online.hpp:294-301
inline void fresh_h_init(const double* v, int64_t F, const Mat& w, double eps, uint64_t seed, uint64_t t,
                         double* h) {
  const double scale = std::max(mean(v, F), eps) / (double(w.c) * mean(w.d.data(), w.size()));
  auto rng = make_engine(mix_seed(seed, t));
  for (int64_t k = 0; k < w.c; ++k) h[k] = scale * uniform_open01(rng);
}

// online.hpp:303-309
inline double smoothed_divergence_to(const double* v, const double* approx_plus_eps, int64_t F, double eps) {
  double acc = 0.0;
  for (int64_t i = 0; i < F; ++i) acc += is_term((v[i] + eps - approx_plus_eps[i]) / approx_plus_eps[i]);
  return acc;
}

// online.hpp:318-337 — rho scales the PAST statistics.
inline void dictionary_commit(Online& st) {
  for (int64_t i = 0; i < st.a.size(); ++i) {
    st.a.d[size_t(i)] = st.rho * st.a.d[size_t(i)] + st.pending_a.d[size_t(i)];
    st.b.d[size_t(i)] = st.rho * st.b.d[size_t(i)] + st.pending_b.d[size_t(i)];
  }
  const Mat w_old = st.w;
  st.w = update_w(st.a, st.b, w_old);
  if (!all_finite(st.w))
    throw Error(NUMERICAL_FAILURE, "online: non-finite dictionary update at t = " + std::to_string(st.t));
  rescale_dictionary(st.w, st.a, st.b, st.restart == Restart::warm ? &st.warm_h : nullptr);
  st.last_delta = frobenius_delta(st.w, w_old);
  std::fill(st.pending_a.d.begin(), st.pending_a.d.end(), 0.0);
  std::fill(st.pending_b.d.begin(), st.pending_b.d.end(), 0.0);
  st.last_minibatch_obj = st.pending_count ? st.pending_div / double(st.pending_count) : 0.0;
  st.pending_div = 0.0;
  st.pending_count = 0;
  ++st.commits;
}

// online.hpp:342-368 — one sample (frame v of length F, dataset index idx).
inline void online_step(Online& st, const double* v, int64_t F, uint64_t idx, const Config& cfg) {
  if (F != st.w.r) throw Error(SHAPE_MISMATCH, "online_step: frame size vs dictionary rows");
  const double eps = cfg.epsilon;
  const int iters = cfg.effective_inner_iters();
  const int64_t K = st.w.c;
  st.scratch_h.resize(size_t(K));
  if (st.restart == Restart::warm) {
    if (int64_t(idx) >= st.warm_h.c) throw Error(SHAPE_MISMATCH, "online_step: sample index outside warm activation store");
    std::copy(st.warm_h.col(int64_t(idx)), st.warm_h.col(int64_t(idx)) + K, st.scratch_h.begin());
  } else {
    fresh_h_init(v, F, st.w, eps, st.seed, st.t, st.scratch_h.data());
  }
  for (int64_t k = 0; k < K; ++k)
    if (st.scratch_h[size_t(k)] <= 0.0) throw Error(NON_POSITIVE_INIT, "solve_h: h0 must be positive");
  solve_h(v, st.w, st.scratch_h.data(), iters, eps, st.scratch_approx, st.scratch_ratio);
  if (st.restart == Restart::warm) std::copy(st.scratch_h.begin(), st.scratch_h.end(), st.warm_h.col(int64_t(idx)));
  accumulate_sample_stats(v, st.w, st.scratch_h.data(), eps, st.pending_a, st.pending_b, st.scratch_approx);
  st.pending_div += smoothed_divergence_to(v, st.scratch_approx.data(), F, eps);
  st.pending_count += 1;
  st.t += 1;
  if (st.t % uint64_t(cfg.beta) == 0) dictionary_commit(st);
}

// online.hpp:375-407 without the wall clock: frames come from `next(t)` which
// returns (pointer to F doubles, index) or nullptr at end of source.
template <class Next>
inline void online_resume(Online& st, Next&& next, const Config& cfg) {
  cfg.validate();
  const uint64_t budget = cfg.max_epochs_or_samples;
  const double eta = cfg.effective_eta(st.w.r, st.w.c);
  bool stop = false;
  while (!stop) {
    if (st.t >= budget) break;
    uint64_t idx = 0;
    const double* v = next(idx);
    if (!v) break;
    online_step(st, v, st.w.r, idx, cfg);
    if (st.t % uint64_t(cfg.beta) == 0) {
      st.trace.push_back({st.t, st.last_minibatch_obj});
      if (eta > 0.0 && st.last_delta < eta) stop = true;
    }
  }
  if (st.trace.empty() && st.pending_count > 0)
    st.trace.push_back({st.t, st.pending_div / double(st.pending_count)});
  if (!st.trace.empty()) st.final_train_obj = st.trace.back().train_obj;
}

// ---- batch trainer (reference batch.hpp:84-143) --------------------------------
struct Batch {
  Mat w, h;
  uint64_t epoch = 0;
  double last_delta = 0.0;
  std::vector<double> obj;  // per-epoch objective trace
  double initial_obj = 0.0;
  double final_train_obj = 0.0;
};

inline Batch batch_train(const Mat& v, const Config& cfg, const Mat& w0, const Mat& h0) {
  cfg.validate();
  if (v.c == 0) throw Error(EMPTY_DATASET, "batch_train: empty dataset");
  if (w0.r != v.r || h0.c != v.c || h0.r != w0.c) throw Error(SHAPE_MISMATCH, "batch_train: inconsistent V/W0/H0 shapes");
  for (double x : w0.d)
    if (x <= 0.0) throw Error(NON_POSITIVE_INIT, "batch_train: w0 and h0 must be strictly positive");
  for (double x : h0.d)
    if (x <= 0.0) throw Error(NON_POSITIVE_INIT, "batch_train: w0 and h0 must be strictly positive");
  const double eps = cfg.epsilon;
  const double eta = cfg.effective_eta(w0.r, w0.c);
  const int64_t F = v.r, K = w0.c, N = v.c;
  Batch st;
  st.w = w0;
  st.h = h0;
  double prev = objective(v, st.w, st.h, eps);
  st.initial_obj = prev;
  std::vector<double> ap(static_cast<size_t>(F)), q(static_cast<size_t>(F)), r(static_cast<size_t>(F));
  for (uint64_t epoch = 1; epoch <= cfg.max_epochs_or_samples; ++epoch) {
    // batch.hpp:110-115 — one multiplicative pass over H at fixed W
    for (int64_t n = 0; n < N; ++n) {
      double* hn = st.h.col(n);
      gemv(st.w, hn, ap.data());
      const double* pv = v.col(n);
      for (int64_t f = 0; f < F; ++f) {
        const double x = ap[f] + eps;
        q[f] = (pv[f] + eps) / (x * x);
        r[f] = 1.0 / x;
      }
      for (int64_t k = 0; k < K; ++k) {
        const double* wk = st.w.col(k);
        double nu = 0.0, de = 0.0;
        for (int64_t f = 0; f < F; ++f) {
          nu += wk[f] * q[f];
          de += wk[f] * r[f];
        }
        hn[k] *= std::sqrt(nu / de);
      }
    }
    Mat a, b;
    batch_stats(v, st.w, st.h, eps, a, b);  // batch.hpp:117
    Mat wn = update_w(a, b, st.w);          // batch.hpp:118-119
    if (!all_finite(wn)) throw Error(NUMERICAL_FAILURE, "batch_train: non-finite dictionary update");
    rescale_dictionary(wn, a, b, &st.h);  // batch.hpp:122
    st.last_delta = frobenius_delta(wn, st.w);
    st.w = wn;
    st.epoch = epoch;
    const double obj = objective(v, st.w, st.h, eps);  // batch.hpp:128
    if (obj > prev + 1e-6 * prev + 1e-15)
      throw Error(DIVERGED_OBJECTIVE, "batch_train: objective increased at epoch " + std::to_string(epoch));
    prev = obj;
    st.obj.push_back(obj);
    if (st.last_delta < eta) break;
  }
  st.final_train_obj = prev;
  return st;
}

}  // namespace isnmf_oracle
