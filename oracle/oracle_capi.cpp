// TEST INFRASTRUCTURE ONLY — extern "C" face of the CPU fp64 oracle
// (isnmf_oracle.hpp) for the Python tests and bench.py's CPU arm.
// Every entry returns 0 or an isnmf_oracle::Code; the message of the last
// failure is available from oracle_last_error().
#include <atomic>
#include <cstring>
#include <memory>
#include <thread>

#include "isnmf_oracle.hpp"

using namespace isnmf_oracle;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

Mat wrap(const double* p, int64_t r, int64_t c) {
  Mat m(r, c);
  if (r * c > 0) std::memcpy(m.d.data(), p, sizeof(double) * size_t(r * c));
  return m;
}
void unwrap(const Mat& m, double* p) {
  if (m.size()) std::memcpy(p, m.d.data(), sizeof(double) * size_t(m.size()));
}

Config make_cfg(int k, double eps, double eta, int beta, double r, int inner_iters, int restart, uint64_t seed,
                uint64_t budget, double delta) {
  Config c;
  c.k = k;
  c.epsilon = eps;
  c.eta = eta;
  c.beta = beta;
  c.r = r;
  c.inner_iters = inner_iters;
  c.restart = restart == 0 ? Restart::warm : Restart::fresh;
  c.seed = seed;
  c.max_epochs_or_samples = budget;
  c.init_stats_weight = delta;
  return c;
}
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

// ---- rng ----
uint64_t oracle_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t oracle_mix_seed(uint64_t s, uint64_t t) { return mix_seed(s, t); }
void oracle_uniform01(uint64_t seed, int64_t n, double* out) {
  auto g = make_engine(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = uniform01(g);
}
void oracle_cycle_permutation(uint64_t seed, uint64_t cycle, uint64_t n, uint64_t* out) {
  auto p = cycle_permutation(seed, cycle, n);
  std::memcpy(out, p.data(), sizeof(uint64_t) * p.size());
}

// ---- kernels ----
int oracle_is_divergence(const double* y, int64_t ny, const double* x, int64_t nx, double eps, double* out) {
  return guard([&] { *out = is_divergence(y, x, ny, nx, eps); });
}
int oracle_objective(const double* v, const double* w, const double* h, int64_t F, int64_t K, int64_t N, double eps,
                     double* out) {
  return guard([&] { *out = objective(wrap(v, F, N), wrap(w, F, K), wrap(h, K, N), eps); });
}
// Solves every column of V (F x N) from h0 (K x N) independently.
int oracle_solve_h(const double* v, const double* w, const double* h0, int64_t F, int64_t K, int64_t N, int iters,
                   double eps, double* h_out) {
  return guard([&] {
    Mat W = wrap(w, F, K);
    for (int64_t n = 0; n < N; ++n) solve_h_checked(v + n * F, F, W, h0 + n * K, K, iters, eps, h_out + n * K);
  });
}
// kernels.hpp:112-121 summed over the N columns in order.
int oracle_sample_stats(const double* v, const double* w, const double* h, int64_t F, int64_t K, int64_t N,
                        double eps, double* a, double* b) {
  return guard([&] {
    require_epsilon(eps);
    Mat W = wrap(w, F, K), A(F, K), B(F, K);
    std::vector<double> ap;
    for (int64_t n = 0; n < N; ++n) accumulate_sample_stats(v + n * F, W, h + n * K, eps, A, B, ap);
    unwrap(A, a);
    unwrap(B, b);
  });
}
int oracle_batch_stats(const double* v, const double* w, const double* h, int64_t F, int64_t K, int64_t N,
                       double eps, double* a, double* b) {
  return guard([&] {
    Mat A, B;
    batch_stats(wrap(v, F, N), wrap(w, F, K), wrap(h, K, N), eps, A, B);
    unwrap(A, a);
    unwrap(B, b);
  });
}
int oracle_update_w(const double* a, const double* b, const double* wp, int64_t F, int64_t K, double* w) {
  return guard([&] { unwrap(update_w(wrap(a, F, K), wrap(b, F, K), wrap(wp, F, K)), w); });
}
int oracle_aux_value(const double* a, const double* b, const double* w, int64_t F, int64_t K, double* out) {
  return guard([&] { *out = aux_value(wrap(a, F, K), wrap(b, F, K), wrap(w, F, K)); });
}
int oracle_aux_constant(const double* v, const double* w, const double* h, int64_t F, int64_t K, int64_t N, double eps,
                        double* out) {
  return guard([&] { *out = aux_constant(wrap(v, F, N), wrap(w, F, K), wrap(h, K, N), eps); });
}
int oracle_rescale_dictionary(double* w, double* a, double* b, int64_t F, int64_t K, double* warm_h, int64_t N) {
  return guard([&] {
    Mat W = wrap(w, F, K), A = wrap(a, F, K), B = wrap(b, F, K);
    Mat H = warm_h ? wrap(warm_h, K, N) : Mat();
    rescale_dictionary(W, A, B, warm_h ? &H : nullptr);
    unwrap(W, w);
    unwrap(A, a);
    unwrap(B, b);
    if (warm_h) unwrap(H, warm_h);
  });
}
int oracle_frobenius_delta(const double* a, int64_t ar, int64_t ac, const double* b, int64_t br, int64_t bc,
                           double* out) {
  return guard([&] { *out = frobenius_delta(wrap(a, ar, ac), wrap(b, br, bc)); });
}
int oracle_config_check(int k, double eps, double eta, int beta, double r, int inner_iters, int restart, int n_seeds,
                        double delta, int64_t F, int64_t K, int* eff_iters, double* eff_eta) {
  return guard([&] {
    Config c = make_cfg(k, eps, eta, beta, r, inner_iters, restart, 1, 500, delta);
    c.n_seeds = n_seeds;
    c.validate();
    *eff_iters = c.effective_inner_iters();
    *eff_eta = c.effective_eta(F, K);
  });
}
int oracle_fresh_h_init(const double* v, const double* w, int64_t F, int64_t K, double eps, uint64_t seed, uint64_t t,
                        double* h) {
  return guard([&] { fresh_h_init(v, F, wrap(w, F, K), eps, seed, t, h); });
}
int oracle_init_from_samples(const double* v, int64_t F, int64_t N, int k, uint64_t seed, double eps, double* w) {
  return guard([&] { unwrap(init_from_samples(wrap(v, F, N), k, seed, eps), w); });
}
int oracle_default_h0(const double* v, const double* w, int64_t F, int64_t K, int64_t N, double eps, double* h) {
  return guard([&] { unwrap(default_h0(wrap(v, F, N), wrap(w, F, K), eps), h); });
}

int oracle_evaluate_heldout(const double* w, const double* test, int64_t F, int64_t K, int64_t Ft, int64_t N,
                            double eps, int iters, uint64_t seed, double* out) {
  return guard([&] { *out = evaluate_heldout(wrap(w, F, K), wrap(test, Ft, N), eps, iters, seed); });
}
int oracle_heldout_h0(const double* w, const double* test, int64_t F, int64_t K, int64_t N, double eps, uint64_t seed,
                      double* h) {
  return guard([&] { unwrap(heldout_h0(wrap(w, F, K), wrap(test, F, N), eps, seed), h); });
}

// ---- online trainer ----
struct OracleOnline {
  Online st;
  Config cfg;
};

// restart: 0 warm, 1 fresh.  dataset (F x N fp64) only needed for warm; sized
// selects rho = r^(beta/N) (online.hpp:274-277).
int oracle_online_create(OracleOnline** out, const double* w0, int64_t F, int64_t K, int beta, double r,
                         int inner_iters, int restart, uint64_t seed, double eps, double eta, uint64_t budget,
                         double delta, int sized, uint64_t dataset_size, const double* dataset, int64_t N) {
  return guard([&] {
    auto o = std::make_unique<OracleOnline>();
    o->cfg = make_cfg(int(K), eps, eta, beta, r, inner_iters, restart, seed, budget, delta);
    Mat ds = dataset ? wrap(dataset, F, N) : Mat();
    o->st = make_online_state(wrap(w0, F, K), o->cfg, sized != 0, dataset_size, dataset ? &ds : nullptr);
    *out = o.release();
  });
}
void oracle_online_destroy(OracleOnline* o) { delete o; }

// Overwrites state fields (NULL pointers keep the current value).
int oracle_online_set(OracleOnline* o, const double* w, const double* a, const double* b, const double* pa,
                      const double* pb, const double* warm_h, int64_t warm_n, double rho, uint64_t t,
                      uint64_t commits) {
  return guard([&] {
    const int64_t F = o->st.w.r, K = o->st.w.c;
    if (w) o->st.w = wrap(w, F, K);
    if (a) o->st.a = wrap(a, F, K);
    if (b) o->st.b = wrap(b, F, K);
    if (pa) o->st.pending_a = wrap(pa, F, K);
    if (pb) o->st.pending_b = wrap(pb, F, K);
    if (warm_h) o->st.warm_h = wrap(warm_h, K, warm_n);
    if (rho >= 0.0) o->st.rho = rho;
    o->st.t = t;
    o->st.commits = commits;
  });
}

int oracle_online_get(OracleOnline* o, double* w, double* a, double* b, double* pa, double* pb, double* warm_h,
                      uint64_t* t, uint64_t* commits, double* scalars /* last_delta, last_obj, pending_div,
                      pending_count, rho, final_train_obj */) {
  return guard([&] {
    if (w) unwrap(o->st.w, w);
    if (a) unwrap(o->st.a, a);
    if (b) unwrap(o->st.b, b);
    if (pa) unwrap(o->st.pending_a, pa);
    if (pb) unwrap(o->st.pending_b, pb);
    if (warm_h) unwrap(o->st.warm_h, warm_h);
    if (t) *t = o->st.t;
    if (commits) *commits = o->st.commits;
    if (scalars) {
      scalars[0] = o->st.last_delta;
      scalars[1] = o->st.last_minibatch_obj;
      scalars[2] = o->st.pending_div;
      scalars[3] = double(o->st.pending_count);
      scalars[4] = o->st.rho;
      scalars[5] = o->st.final_train_obj;
    }
  });
}

// online_resume (online.hpp:375-407) over frames v (F x n, fp32 or fp64 via
// is_f32) visited in order with dataset indices idx (NULL = 0..n-1 offset by
// index_base).  Trace points (samples, train_obj) are appended to the arrays.
int oracle_online_run(OracleOnline* o, const void* v, int is_f32, int64_t n, const uint64_t* idx, uint64_t index_base,
                      uint64_t* trace_t, double* trace_obj, int64_t trace_cap, int64_t* n_trace) {
  return guard([&] {
    const int64_t F = o->st.w.r;
    std::vector<double> frame(static_cast<size_t>(F));
    int64_t pos = 0;
    const size_t before = o->st.trace.size();
    auto next = [&](uint64_t& index) -> const double* {
      if (pos >= n) return nullptr;
      if (is_f32) {
        const float* p = static_cast<const float*>(v) + pos * F;
        for (int64_t f = 0; f < F; ++f) frame[size_t(f)] = double(p[f]);
      } else {
        const double* p = static_cast<const double*>(v) + pos * F;
        std::copy(p, p + F, frame.begin());
      }
      index = idx ? idx[pos] : index_base + uint64_t(pos);
      ++pos;
      return frame.data();
    };
    online_resume(o->st, next, o->cfg);
    int64_t m = 0;
    for (size_t i = before; i < o->st.trace.size() && m < trace_cap; ++i, ++m) {
      if (trace_t) trace_t[m] = o->st.trace[i].samples;
      if (trace_obj) trace_obj[m] = o->st.trace[i].train_obj;
    }
    if (n_trace) *n_trace = m;
  });
}

// One sample through online_step (online.hpp:342-368).
int oracle_online_step(OracleOnline* o, const double* v, int64_t F, uint64_t index) {
  return guard([&] { online_step(o->st, v, F, index, o->cfg); });
}
int oracle_online_commit(OracleOnline* o) {
  return guard([&] { dictionary_commit(o->st); });
}

// ---- batch trainer ----
int oracle_batch_train(const double* v, const double* w0, const double* h0, int64_t F, int64_t K, int64_t N,
                       uint64_t max_epochs, double eps, double eta, double* w_out, double* h_out, double* obj_trace,
                       int64_t* epochs, double* initial_obj, double* last_delta) {
  return guard([&] {
    Config c = make_cfg(int(K), eps, eta, 1000, 0.7, 0, 0, 1, max_epochs, 1.0);
    Batch bt = batch_train(wrap(v, F, N), c, wrap(w0, F, K), wrap(h0, K, N));
    unwrap(bt.w, w_out);
    unwrap(bt.h, h_out);
    for (size_t i = 0; i < bt.obj.size(); ++i) obj_trace[i] = bt.obj[i];
    *epochs = int64_t(bt.epoch);
    *initial_obj = bt.initial_obj;
    *last_delta = bt.last_delta;
  });
}

// ---- CPU baseline: online mini-batches with the per-frame H solves of each
// mini-batch split across `threads` host threads (SPEC.md:290 permits it);
// stats of each thread's contiguous frame range are summed in thread order.
// Warm store of ones semantics (h0 = cumulative rescale products), fp32 V.
int oracle_baseline_online(const float* v, int64_t F, int64_t K, int64_t n_frames, int beta, int iters, double eps,
                           double rho, const double* w0, const double* a0, const double* b0, int threads,
                           double* w_out, double* obj_out) {
  return guard([&] {
    Mat W = wrap(w0, F, K), A = wrap(a0, F, K), B = wrap(b0, F, K);
    std::vector<double> hscale(size_t(K), 1.0);  // warm_h = ones, rescaled per commit
    const int T = std::max(1, threads);
    std::vector<Mat> pa(size_t(T), Mat(F, K)), pb(size_t(T), Mat(F, K));
    std::vector<double> pdiv(static_cast<size_t>(T));
    double last_obj = 0.0;
    for (int64_t start = 0; start + beta <= n_frames; start += beta) {
      auto work = [&](int tid) {
        const int64_t lo = start + beta * tid / T, hi = start + beta * (tid + 1) / T;
        std::fill(pa[size_t(tid)].d.begin(), pa[size_t(tid)].d.end(), 0.0);
        std::fill(pb[size_t(tid)].d.begin(), pb[size_t(tid)].d.end(), 0.0);
        pdiv[size_t(tid)] = 0.0;
        std::vector<double> fr(static_cast<size_t>(F)), h(static_cast<size_t>(K)), ap, rt;
        for (int64_t n = lo; n < hi; ++n) {
          for (int64_t f = 0; f < F; ++f) fr[size_t(f)] = double(v[n * F + f]);
          h = hscale;
          solve_h(fr.data(), W, h.data(), iters, eps, ap, rt);
          accumulate_sample_stats(fr.data(), W, h.data(), eps, pa[size_t(tid)], pb[size_t(tid)], ap);
          pdiv[size_t(tid)] += smoothed_divergence_to(fr.data(), ap.data(), F, eps);
        }
      };
      std::vector<std::thread> pool;
      for (int tid = 1; tid < T; ++tid) pool.emplace_back(work, tid);
      work(0);
      for (auto& th : pool) th.join();
      double dsum = 0.0;
      for (int tid = 0; tid < T; ++tid) {
        for (int64_t i = 0; i < A.size(); ++i) {
          A.d[size_t(i)] = (tid == 0 ? rho * A.d[size_t(i)] : A.d[size_t(i)]) + pa[size_t(tid)].d[size_t(i)];
          B.d[size_t(i)] = (tid == 0 ? rho * B.d[size_t(i)] : B.d[size_t(i)]) + pb[size_t(tid)].d[size_t(i)];
        }
        dsum += pdiv[size_t(tid)];
      }
      Mat w_old = W;
      W = update_w(A, B, w_old);
      if (!all_finite(W)) throw Error(NUMERICAL_FAILURE, "baseline: non-finite W");
      for (int64_t k = 0; k < K; ++k) {
        double s = 0.0;
        for (int64_t f = 0; f < F; ++f) s += W(f, k);
        if (!(s > 0.0)) throw Error(ZERO_COLUMN, "baseline: dead atom");
        for (int64_t f = 0; f < F; ++f) {
          W(f, k) /= s;
          A(f, k) /= s;
          B(f, k) *= s;
        }
        hscale[size_t(k)] *= s;
      }
      last_obj = dsum / double(beta);
    }
    unwrap(W, w_out);
    *obj_out = last_obj;
  });
}

}  // extern "C"
