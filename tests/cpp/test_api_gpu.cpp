// The reference's own unit tests (proj/tests/test_kernels.cpp, test_core.cpp
// rescale cases) restated against the isnmf-b200 C++ API, which computes on the
// B200 in fp32: tolerances that the reference states for fp64 are widened to
// the fp32 level and marked; plus trainer-level checks of online_train /
// online_resume / batch_train through the same API.
#include <sstream>

#include "isnmf/isnmf.hpp"
#include "minitest.hpp"

using namespace isnmf;

static Matrix random_positive(Index rows, Index cols, std::uint64_t seed, double lo = 0.05, double hi = 2.0) {
  auto rng = make_engine(seed);
  Matrix m(rows, cols);
  for (Index j = 0; j < cols; ++j)
    for (Index i = 0; i < rows; ++i) m(i, j) = lo + (hi - lo) * uniform01(rng);
  return m;
}
static Vector random_positive_vec(Index n, std::uint64_t seed, double lo = 0.05, double hi = 2.0) {
  return random_positive(n, 1, seed, lo, hi).col(0);
}
static Matrix elementwise_sqrt_ratio(const Matrix& a, const Matrix& b) {
  Matrix r(a.rows(), a.cols());
  for (Index i = 0; i < a.size(); ++i) r.data()[i] = std::sqrt(a.data()[i] / b.data()[i]);
  return r;
}

TEST_CASE("is_divergence values and properties (test_kernels.cpp:28-77)") {
  const double eps = 1e-12;
  Vector y = random_positive_vec(16, 1);
  CHECK(is_divergence(y, y, eps) == 0.0);
  Vector x = y;
  x[3] *= 1.5;
  CHECK(is_divergence(y, x, eps) > 0.0);
  CHECK_REL(is_divergence(Vector::Constant(2, 1.0), Vector::Constant(2, 2.0), 1e-15), 2.0 * (0.5 + std::log(2.0) - 1.0),
            1e-9);
  auto rng = make_engine(7);
  for (int trial = 0; trial < 50; ++trial) {
    Vector a = random_positive_vec(8, 100 + trial), b = random_positive_vec(8, 200 + trial);
    const double lambda = 0.01 + 100.0 * uniform01(rng);
    Vector la = a, lb = b;
    for (Index i = 0; i < 8; ++i) la[i] *= lambda, lb[i] *= lambda;
    CHECK_REL(is_divergence(la, lb, lambda * 1e-9), is_divergence(a, b, 1e-9), 1e-10);
  }
  CHECK_THROWS_AS(is_divergence(Vector::Ones(3), Vector::Ones(4), eps), ShapeMismatch);
  Vector neg = Vector::Ones(3);
  neg[0] = -0.5;
  CHECK_THROWS_AS(is_divergence(neg, neg, eps), NegativeInput);
  CHECK_THROWS_AS(is_divergence(Vector::Ones(3), Vector::Ones(3), 0.0), NegativeInput);
}

TEST_CASE("solve_h descends and finds optima (test_kernels.cpp:79-131)") {
  const double eps = 1e-12;
  Matrix w = random_positive(6, 2, 11);
  Vector h_star = random_positive_vec(2, 12);
  Vector h = solve_h(w * h_star, w, h_star, 25, 1e-14);
  for (Index k = 0; k < 2; ++k) CHECK(std::abs(h[k] - h_star[k]) < 1e-5);  // reference: 1e-9 (fp64)
  Matrix w1 = Matrix::Constant(1, 1, 2.0);
  Vector h1 = solve_h(Vector::Constant(1, 4.0), w1, Vector::Constant(1, 0.3), 100, eps);
  CHECK(std::abs(h1[0] - 2.0) < 1e-5);  // reference: 1e-6
  Matrix w9 = random_positive(9, 3, 13);
  Vector v9 = random_positive_vec(9, 14);
  Vector hh = random_positive_vec(3, 15);
  double prev = is_divergence(v9, w9 * hh, eps);
  for (int it = 0; it < 60; ++it) {
    hh = solve_h(v9, w9, hh, 1, eps);
    const double cur = is_divergence(v9, w9 * hh, eps);
    CHECK(cur <= prev * (1.0 + 1e-6) + 1e-10);  // reference: + 1e-10 (fp64)
    prev = cur;
  }
  CHECK_THROWS_AS(solve_h(random_positive_vec(3, 17), random_positive(3, 2, 16), Vector::Zero(2), 5, eps),
                  NonPositiveInit);
}

TEST_CASE("sample statistics (test_kernels.cpp:133-165)") {
  SampleStats s = sample_stats(Vector::Constant(1, 8.0), Matrix::Constant(1, 1, 2.0), Vector::Constant(1, 1.0), 1e-30);
  CHECK_REL(s.a(0, 0), 8.0, 1e-6);
  CHECK_REL(s.b(0, 0), 0.5, 1e-6);
  SampleStats s1 = sample_stats(Vector::Constant(1, 0.0), Matrix::Constant(1, 1, 1.0), Vector::Constant(1, 1.0), 1.0);
  CHECK_REL(s1.a(0, 0), 0.25, 1e-6);
  CHECK_REL(s1.b(0, 0), 0.5, 1e-6);
  Matrix w = random_positive(7, 3, 21);
  Vector h = random_positive_vec(3, 22);
  SampleStats s2 = sample_stats(w * h, w, h, 1e-30);
  CHECK((elementwise_sqrt_ratio(s2.a, s2.b) - w).maxAbs() < 1e-5);  // reference: 1e-10
}

TEST_CASE("batch statistics agree with per-sample sums (test_kernels.cpp:167-198)") {
  const double eps = 1e-12;
  Matrix v = random_positive(6, 9, 31), w = random_positive(6, 3, 32), h = random_positive(3, 9, 33);
  SampleStats full = batch_stats(v, w, h, eps);
  Matrix sa = Matrix::Zero(6, 3), sb = Matrix::Zero(6, 3);
  for (Index n = 0; n < 9; ++n) {
    SampleStats s = sample_stats(v.col(n), w, h.col(n), eps);
    sa = sa + s.a;
    sb = sb + s.b;
  }
  for (Index i = 0; i < sa.size(); ++i) {
    CHECK_REL(full.a.data()[i], sa.data()[i], 1e-5);  // reference: 1e-10
    CHECK_REL(full.b.data()[i], sb.data()[i], 1e-5);
  }
  SampleStats ex = batch_stats(w * h, w, h, 1e-30);
  CHECK((elementwise_sqrt_ratio(ex.a, ex.b) - w).maxAbs() < 1e-5);
}

TEST_CASE("update_w is the auxiliary argmin (test_kernels.cpp:200-259)") {
  Matrix a = Matrix::Constant(3, 2, 0.7);
  CHECK((update_w(a, a, Matrix::Constant(3, 2, 0.123)) - Matrix::Ones(3, 2)).maxAbs() < 1e-15);
  CHECK_REL(update_w(Matrix::Constant(1, 1, 4.0), Matrix::Constant(1, 1, 1.0), Matrix::Ones(1, 1))(0, 0), 2.0, 1e-15);
  Matrix a2 = Matrix::Zero(2, 1), b2 = Matrix::Zero(2, 1), prev(2, 1);
  prev(0, 0) = 0.3;
  prev(1, 0) = 0.7;
  a2(0, 0) = 1.0;
  b2(0, 0) = 4.0;
  Matrix w2 = update_w(a2, b2, prev);
  CHECK_REL(w2(0, 0), 0.5, 1e-15);
  CHECK(w2(1, 0) == 0.7);
  CHECK_THROWS_AS(update_w(Matrix::Ones(1, 1), Matrix::Zero(1, 1), Matrix::Ones(1, 1)), InconsistentStats);
  auto rng = make_engine(55);
  for (int trial = 0; trial < 20; ++trial) {
    Matrix at = random_positive(4, 3, 700 + trial), bt = random_positive(4, 3, 800 + trial);
    Matrix wt = update_w(at, bt, Matrix::Ones(4, 3));
    const double base = aux_value(at, bt, wt);
    for (int probe = 0; probe < 10; ++probe) {
      const Index i = Index(uniform_below(rng, 4)), j = Index(uniform_below(rng, 3));
      Matrix wp = wt;
      wp(i, j) *= uniform01(rng) < 0.5 ? 1.01 : 0.99;
      CHECK(aux_value(at, bt, wp) > base);
    }
  }
}

TEST_CASE("auxiliary function majorizes the objective (test_kernels.cpp:261-303)") {
  Matrix one = Matrix::Ones(1, 1);
  CHECK_REL(aux_value(one, one, one), 2.0, 1e-15);
  Matrix w = random_positive(5, 2, 61), h = random_positive(2, 7, 62);
  CHECK(objective(w * h, w, h, 1e-30) < 1e-6);  // reference: 1e-12 (fp64 reconstruction)
  const double eps = 1e-12;
  for (int trial = 0; trial < 10; ++trial) {
    const Index f = 8, k = 3, n = 6;
    Matrix v = random_positive(f, n, 1000 + trial), wu = random_positive(f, k, 1100 + trial),
           hh = random_positive(k, n, 1200 + trial);
    SampleStats s = batch_stats(v, wu, hh, eps);
    const double c = aux_constant(v, wu, hh, eps);
    const double n_obj = double(n) * objective(v, wu, hh, eps);
    CHECK_REL(aux_value(s.a, s.b, wu) + c, n_obj, 1e-5);  // reference: 1e-8
    for (int probe = 0; probe < 30; ++probe) {
      Matrix wp = random_positive(f, k, 2000 + 100 * trial + probe, 0.02, 3.0);
      CHECK(aux_value(s.a, s.b, wp) + c >= double(n) * objective(v, wp, hh, eps) * (1 - 1e-5));
    }
  }
}

TEST_CASE("rescale_dictionary normalizes and compensates (test_core.cpp:47-101)") {
  Dictionary d1{Matrix::Constant(2, 1, 2.0), Matrix::Constant(2, 1, 1.0), Matrix::Constant(2, 1, 1.0)};
  rescale_dictionary(d1);
  CHECK(std::abs(d1.w(0, 0) - 0.5) < 1e-15 && std::abs(d1.a(1, 0) - 0.25) < 1e-15 && d1.b(0, 0) == 4.0);
  Matrix w = random_positive(6, 3, 2), h = random_positive(3, 5, 3);
  Matrix product = w * h;
  Dictionary d2{w, random_positive(6, 3, 4), random_positive(6, 3, 5)};
  rescale_dictionary(d2, &h);
  CHECK((d2.w * h - product).norm() < 1e-12);
  Dictionary d3{random_positive(5, 2, 6), random_positive(5, 2, 7), random_positive(5, 2, 8)};
  rescale_dictionary(d3);
  Dictionary again = d3;
  rescale_dictionary(again);
  CHECK((again.w - d3.w).maxAbs() < 1e-12 && (again.b - d3.b).maxAbs() < 1e-12);
  Dictionary dead{Matrix::Zero(3, 1), Matrix::Zero(3, 1), Matrix::Zero(3, 1)};
  CHECK_THROWS_AS(rescale_dictionary(dead), ZeroColumn);
}

static Matrix spectrogram(Index F, Index K, Index N, std::uint64_t seed) {
  Matrix ws = random_positive(F, K, seed, 0.1, 1.0), hs = random_positive(K, N, seed + 1, 0.0, 1.0);
  for (Index i = 0; i < hs.size(); ++i) hs.data()[i] = hs.data()[i] * hs.data()[i] * 2.0;  // sparse-ish
  Matrix v = ws * hs;
  auto rng = make_engine(seed + 2);
  for (Index i = 0; i < v.size(); ++i) v.data()[i] = v.data()[i] * -std::log(uniform_open01(rng)) + 1e-9;
  return v;
}

static Matrix normalized(Matrix w) {
  for (Index k = 0; k < w.cols(); ++k) {
    double s = 0.0;
    for (Index f = 0; f < w.rows(); ++f) s += w(f, k);
    for (Index f = 0; f < w.rows(); ++f) w(f, k) /= s;
  }
  return w;
}

TEST_CASE("online_train over a CyclingSource: trace, budget, warm store (online.hpp:375-419)") {
  const Index F = 65, K = 4, N = 96;
  Matrix v = spectrogram(F, K, N, 9);
  SolverConfig c;
  c.k = int(K);
  c.beta = 16;
  c.r = 0.7;
  c.inner_iters = 3;
  c.eta = 0.0;
  c.max_epochs_or_samples = 3 * N + 5;
  CyclingSource src(v, 4);
  OnlineState st = online_train(src, c, normalized(random_positive(F, K, 5, 0.1, 1.0)));
  CHECK(st.t == 3 * N + 5 && st.commits == (3 * N + 5) / 16 && st.pending_count == (3 * N + 5) % 16);
  CHECK(st.trace.points.size() == st.commits);
  CHECK(st.trace.points.back().samples == st.commits * 16);
  CHECK(st.trace.final_train_obj == st.trace.points.back().train_obj);
  for (Index k = 0; k < K; ++k) {
    double s = 0.0;
    for (Index f = 0; f < F; ++f) s += st.dict.w(f, k);
    CHECK(std::abs(s - 1.0) < 1e-12);
  }
  CHECK(st.warm_h.rows() == K && st.warm_h.cols() == N && st.warm_h.allFinite());
  // resume continues from t and keeps the source position (exact seek)
  c.max_epochs_or_samples = 4 * N;
  online_resume(st, src, c);
  CHECK(st.t == 4 * N);
}

TEST_CASE("online callbacks see every commit and can stop (online.hpp:390-397)") {
  const Index F = 33, K = 3, N = 64;
  Matrix v = spectrogram(F, K, N, 3);
  SolverConfig c;
  c.k = int(K);
  c.beta = 8;
  c.restart = RestartMode::fresh;
  c.inner_iters = 5;
  c.eta = 0.0;
  c.max_epochs_or_samples = N;
  CyclingSource src(v, 2);
  int calls = 0;
  OnlineState st = online_train(src, c, normalized(random_positive(F, K, 6, 0.1, 1.0)), [&](OnlineState& s) {
    ++calls;
    CHECK(s.t == std::uint64_t(8 * calls) && s.commits == std::uint64_t(calls));
    return calls < 5;
  });
  CHECK(calls == 5 && st.t == 40 && st.trace.points.size() == 5);
}

TEST_CASE("online_step / dictionary_commit per sample (online.hpp:318-368)") {
  const Index F = 17, K = 2;
  Matrix v = spectrogram(F, K, 4, 12);
  SolverConfig c;
  c.k = int(K);
  c.beta = 2;
  c.restart = RestartMode::fresh;
  c.inner_iters = 4;
  OnlineState st = make_online_state(normalized(random_positive(F, K, 2, 0.1, 1.0)), c, 4);
  const Matrix w0 = st.dict.w;
  online_step(st, Sample{v.col(0), 0}, c);
  CHECK(st.commits == 0 && st.t == 1 && frobenius_delta(st.dict.w, w0) == 0.0 && st.pending_a.maxAbs() > 0.0);
  online_step(st, Sample{v.col(1), 1}, c);
  CHECK(st.commits == 1 && st.pending_a.maxAbs() == 0.0 && frobenius_delta(st.dict.w, w0) > 0.0);
  online_step(st, Sample{v.col(2), 2}, c);
  dictionary_commit(st);
  CHECK(st.commits == 2 && st.pending_count == 0);
  CHECK_THROWS_AS(online_step(st, Sample{Vector::Ones(3), 3}, c), ShapeMismatch);
}

TEST_CASE("batch_train descends and equals online at beta = N, r = 0 (SPEC.md:409-413)") {
  const Index F = 20, K = 4, N = 50;
  Matrix v = spectrogram(F, K, N, 21);
  Matrix w0 = normalized(random_positive(F, K, 22, 0.1, 1.0));
  Matrix h0 = default_h0(v, w0);
  SolverConfig c;
  c.k = int(K);
  c.eta = 0.0;
  c.max_epochs_or_samples = 6;
  BatchState b = batch_train(v, c, w0, h0);
  CHECK(b.epoch == 6 && b.trace.points.size() == 6);
  for (size_t i = 1; i < b.trace.points.size(); ++i)
    CHECK(b.trace.points[i].train_obj <= b.trace.points[i - 1].train_obj * (1 + 1e-6));
  int seen = 0;
  BatchState b2 = batch_train(v, c, w0, h0, [&](BatchState& s) { return ++seen < 3 && s.epoch < 6; });
  CHECK(seen == 3 && b2.epoch == 3);
  SolverConfig oc;
  oc.k = int(K);
  oc.beta = int(N);
  oc.r = 0.0;
  oc.inner_iters = 1;
  oc.eta = 0.0;
  oc.init_stats_weight = 0.0;
  oc.max_epochs_or_samples = 6 * N;
  OnlineState st = make_online_state(w0, oc, std::uint64_t(N), &v);
  st.warm_h = h0;
  GeneratorSource identity([&](std::uint64_t i) { return v.col(Index(i % N)); }, 6 * N, N, 1, false);
  // identity order: column index == dataset index when the generator index is reduced mod N
  struct ModSource final : SampleSource {
    GeneratorSource* g;
    Index n;
    std::optional<Sample> next() override {
      auto s = g->next();
      if (s) s->index %= std::uint64_t(n);
      return s;
    }
    void seek(std::uint64_t t) override { g->seek(t); }
    std::optional<std::uint64_t> size() const override { return std::nullopt; }
  } mod;
  mod.g = &identity;
  mod.n = N;
  online_resume(st, mod, oc);
  for (Index i = 0; i < st.dict.w.size(); ++i) CHECK_REL(st.dict.w.data()[i], b.w.data()[i], 1e-4);
}

MT_MAIN()

TEST_CASE("checkpoint/resume at a commit boundary reproduces the uninterrupted run bitwise (SPEC.md:418)") {
  const Index F = 65, K = 4, N = 96;
  Matrix v = spectrogram(F, K, N, 31);
  Matrix w0 = normalized(random_positive(F, K, 32, 0.1, 1.0));
  SolverConfig c;
  c.k = int(K);
  c.beta = 16;
  c.restart = RestartMode::fresh;
  c.inner_iters = 6;
  c.eta = 0.0;
  c.seed = 9;
  c.max_epochs_or_samples = 2 * N;
  CyclingSource full_src(v, 5);
  OnlineState full = online_train(full_src, c, w0);
  // same run, stopped at t = 80 (a commit boundary), saved, reloaded, resumed
  c.max_epochs_or_samples = 80;
  CyclingSource src(v, 5);
  OnlineState half = online_train(src, c, w0);
  std::stringstream ss;
  save_checkpoint(ss, half);
  OnlineState back = load_checkpoint(ss);
  back.trace.config = c;
  c.max_epochs_or_samples = 2 * N;
  online_resume(back, src, c);
  CHECK(back.t == full.t && back.commits == full.commits);
  CHECK(std::memcmp(back.dict.w.data(), full.dict.w.data(), size_t(F * K) * sizeof(double)) == 0);
  CHECK(std::memcmp(back.dict.a.data(), full.dict.a.data(), size_t(F * K) * sizeof(double)) == 0);
  CHECK(std::memcmp(back.dict.b.data(), full.dict.b.data(), size_t(F * K) * sizeof(double)) == 0);
  // mid-mini-batch checkpoint: pending statistics travel in the file; the split
  // launch sums the same frames in another grouping (fp32 partials), so W agrees
  // to the fp32 level rather than bitwise
  c.max_epochs_or_samples = 87;
  CyclingSource src2(v, 5);
  OnlineState mid = online_train(src2, c, w0);
  std::stringstream s2;
  save_checkpoint(s2, mid);
  OnlineState back2 = load_checkpoint(s2);
  c.max_epochs_or_samples = 2 * N;
  online_resume(back2, src2, c);
  CHECK(back2.t == full.t && back2.commits == full.commits);
  double worst = 0.0;
  for (Index i = 0; i < F * K; ++i)
    worst = std::max(worst, std::abs(back2.dict.w.data()[i] - full.dict.w.data()[i]) / full.dict.w.data()[i]);
  CHECK(worst < 1e-5);
}

TEST_CASE("evaluate_heldout: frozen W, deterministic, errors (harness.hpp:17-37)") {
  const Index F = 33, K = 3, N = 40;
  Matrix v = spectrogram(F, K, N, 41);
  Matrix w = normalized(random_positive(F, K, 42, 0.1, 1.0));
  const Matrix w_copy = w;
  const double d1 = evaluate_heldout(w, v, 1e-12);
  const double d2 = evaluate_heldout(w, v, 1e-12);
  CHECK(d1 == d2 && d1 > 0.0 && std::isfinite(d1));
  CHECK(std::memcmp(w.data(), w_copy.data(), size_t(F * K) * sizeof(double)) == 0);
  CHECK(evaluate_heldout(w, v, 1e-12, 100, 7) != d1);           // the seed picks the random init
  CHECK(evaluate_heldout(w, v, 1e-12, 200) <= d1 * (1 + 1e-6));  // more MM iterations never hurt
  CHECK_THROWS_AS(evaluate_heldout(w, Matrix::Ones(F + 1, 4), 1e-12), ShapeMismatch);
  CHECK_THROWS_AS(evaluate_heldout(w, Matrix(F, 0), 1e-12), EmptyDataset);
}

TEST_CASE("stft_power / discard_silence: frame rule, Parseval, order, errors (audio.hpp:121-187)") {
  std::vector<double> x(4000);
  for (std::size_t i = 0; i < x.size(); ++i) x[i] = std::sin(0.05 * double(i)) + (i % 7 == 0 ? 0.3 : 0.0);
  Matrix p = stft_power(x, 512, 256);
  CHECK(p.rows() == 257 && p.cols() == (4000 - 512) / 256 + 1);
  // Parseval on frame 0: sum |X_f|^2 over the full spectrum = W * sum (w x)^2
  double e_time = 0.0;
  for (int i = 0; i < 512; ++i) {
    const double w = std::sin(M_PI * (i + 0.5) / 512) * x[std::size_t(i)];
    e_time += w * w;
  }
  double e_freq = p(0, 0) + p(256, 0);
  for (Index f = 1; f < 256; ++f) e_freq += 2.0 * p(f, 0);
  CHECK_REL(e_freq, 512.0 * e_time, 1e-10);
  CHECK_THROWS_AS(stft_power(x, 511, 256), UnsupportedFormat);
  CHECK_THROWS_AS(stft_power(std::vector<double>(100, 1.0), 512, 256), TooShort);
  Matrix spec = p;
  for (Index f = 0; f < spec.rows(); ++f) spec(f, 3) *= 1e-9;  // -90 dB
  std::vector<FrameMeta> meta(std::size_t(spec.cols()));
  for (std::size_t i = 0; i < meta.size(); ++i) meta[i] = FrameMeta{7, 100 + i};
  SpectrogramDataset ds = discard_silence(spec, -60.0, 16000.0, &meta);
  CHECK(ds.discarded_count == 1 && ds.frames.cols() == spec.cols() - 1 && ds.meta.size() == std::size_t(spec.cols() - 1));
  CHECK(ds.meta[3].frame_index == 104 && ds.frames(10, 3) == spec(10, 4) && ds.sample_rate == 16000.0);
  CHECK_THROWS_AS(discard_silence(Matrix::Zero(4, 5)), AllSilent);
  std::vector<FrameMeta> short_meta(2);
  CHECK_THROWS_AS(discard_silence(spec, -60.0, 0.0, &short_meta), ShapeMismatch);
}
