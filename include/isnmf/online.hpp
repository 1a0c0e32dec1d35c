// isnmf-b200 C++ API — the online IS-NMF trainer (reference
// proj/include/isnmf/online.hpp:24-419): sample sources, OnlineState,
// make_online_state / online_step / dictionary_commit / online_resume /
// online_train, with the same names, signatures, options and exceptions.
//
// The state of record stays in the public fields of OnlineState (host fp64);
// the arithmetic runs in a device engine (C ABI isnmf_online_*): the fields are
// pushed to the engine when a call starts and pulled back when it returns (and
// before every callback).  online_resume pulls frames from the source in blocks
// that end on mini-batch boundaries and hands each block to one engine call;
// without a callback and with eta == 0 it runs up to 64 mini-batches per call.
// warm_h round-trips exactly: the engine's warm activation store is fp64 like the
// reference's (values below fp32's range enter the fp32 solver at a floor that
// leaves W h unchanged and are rescaled back in fp64; kernels.cuh warm_value).
// Checkpointing (save_checkpoint / load_checkpoint, the reference's "ISCK"
// format, online.hpp:421-489) serialises these host fields; see the end of
// this file.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <fstream>
#include <functional>
#include <istream>
#include <limits>
#include <memory>
#include <numeric>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "batch.hpp"
#include "io.hpp"
#include "kernels.hpp"
#include "model.hpp"
#include "report.hpp"
#include "rng.hpp"

namespace isnmf {

/// One frame with its dataset position (the warm activation column).
struct Sample {
  Vector frame;
  std::uint64_t index = 0;
};

/// Frame provider (online.hpp:33-48).
class SampleSource {
 public:
  virtual ~SampleSource() = default;
  virtual std::optional<Sample> next() = 0;
  /// Repositions to global sample ordinal t (seekable sources only).
  virtual void seek(std::uint64_t t) = 0;
  /// Number of distinct frames when finite (rho = r^(beta/N)).
  virtual std::optional<std::uint64_t> size() const = 0;
  /// Whole dataset when in memory (warm restarts need it).
  virtual const Matrix* dataset() const { return nullptr; }
  /// Engine fast path: up to n frames written as fp32 into dst (F floats
  /// each) with their indices; returns the count (0 = end).  The default pulls
  /// through next().
  virtual std::size_t next_block(std::size_t n, Index F, float* dst, std::uint64_t* index) {
    std::size_t m = 0;
    for (; m < n; ++m) {
      auto s = next();
      if (!s) break;
      if (s->frame.size() != F) throw ShapeMismatch("online_step: frame size vs dictionary rows");
      for (Index f = 0; f < F; ++f) dst[size_t(m) * size_t(F) + size_t(f)] = float(s->frame[f]);
      index[m] = s->index;
    }
    return m;
  }
};

namespace detail {
inline std::vector<std::uint64_t> shuffled_range(std::size_t n, std::uint64_t seed, std::uint64_t stream) {
  std::vector<std::uint64_t> p(n);
  std::iota(p.begin(), p.end(), std::uint64_t(0));
  auto rng = make_engine(mix_seed(seed, stream));
  for (std::size_t i = n; i > 1; --i) std::swap(p[i - 1], p[static_cast<std::size_t>(uniform_below(rng, i))]);
  return p;
}
}  // namespace detail

/// Cycles over the columns of an in-memory dataset, re-permuted every cycle
/// by a pure function of (seed, cycle) (online.hpp:53-94).
class CyclingSource final : public SampleSource {
 public:
  CyclingSource(const Matrix& v, std::uint64_t seed) : v_(&v), seed_(seed) {
    if (v.cols() == 0) throw EmptyDataset("CyclingSource: empty dataset");
    load(0);
  }
  std::optional<Sample> next() override {
    if (pos_ == order_.size()) load(cycle_ + 1);
    const std::uint64_t c = order_[pos_++];
    return Sample{v_->col(static_cast<Index>(c)), c};
  }
  std::size_t next_block(std::size_t n, Index F, float* dst, std::uint64_t* index) override {
    if (F != v_->rows()) throw ShapeMismatch("online_step: frame size vs dictionary rows");
    for (std::size_t m = 0; m < n; ++m) {
      if (pos_ == order_.size()) load(cycle_ + 1);
      const std::uint64_t c = order_[pos_++];
      const double* src = v_->col_data(static_cast<Index>(c));
      for (Index f = 0; f < F; ++f) dst[m * size_t(F) + size_t(f)] = float(src[f]);
      index[m] = c;
    }
    return n;
  }
  void seek(std::uint64_t t) override {
    const auto n = static_cast<std::uint64_t>(v_->cols());
    load(t / n);
    pos_ = static_cast<std::size_t>(t % n);
  }
  std::optional<std::uint64_t> size() const override { return static_cast<std::uint64_t>(v_->cols()); }
  const Matrix* dataset() const override { return v_; }

 private:
  void load(std::uint64_t cycle) {
    cycle_ = cycle;
    pos_ = 0;
    order_ = detail::shuffled_range(static_cast<std::size_t>(v_->cols()), seed_, cycle);
  }
  const Matrix* v_;
  std::uint64_t seed_;
  std::uint64_t cycle_ = 0;
  std::size_t pos_ = 0;
  std::vector<std::uint64_t> order_;
};

/// Frames from a deterministic generator, permuted per buffer (online.hpp:98-149).
class GeneratorSource final : public SampleSource {
 public:
  using Generator = std::function<Vector(std::uint64_t)>;
  GeneratorSource(Generator gen, std::optional<std::uint64_t> total, std::size_t buffer_frames, std::uint64_t seed,
                  bool permute = true)
      : gen_(std::move(gen)), total_(total), buffer_(std::max<std::size_t>(1, buffer_frames)), seed_(seed),
        permute_(permute) {}
  std::optional<Sample> next() override {
    if (total_ && t_ >= *total_) return std::nullopt;
    const std::uint64_t block = t_ / buffer_;
    if (block != loaded_ || order_.empty()) load(block);
    const std::uint64_t idx = block * buffer_ + order_[static_cast<std::size_t>(t_ % buffer_)];
    ++t_;
    return Sample{gen_(idx), idx};
  }
  void seek(std::uint64_t t) override { t_ = t; }
  std::optional<std::uint64_t> size() const override { return std::nullopt; }

 private:
  void load(std::uint64_t block) {
    std::size_t len = buffer_;
    if (total_) len = static_cast<std::size_t>(std::min<std::uint64_t>(buffer_, *total_ - block * buffer_));
    if (permute_) {
      order_ = detail::shuffled_range(len, seed_, block);
    } else {
      order_.resize(len);
      std::iota(order_.begin(), order_.end(), std::uint64_t(0));
    }
    loaded_ = block;
  }
  Generator gen_;
  std::optional<std::uint64_t> total_;
  std::size_t buffer_;
  std::uint64_t seed_;
  bool permute_;
  std::uint64_t t_ = 0;
  std::uint64_t loaded_ = ~std::uint64_t(0);
  std::vector<std::uint64_t> order_;
};

/// Headerless chunked wire format [u64 LE count | count x F f64 LE], permuted
/// per buffer; not seekable (online.hpp:151-220).  Frames are decoded into one
/// contiguous fp64 block per buffer (no per-frame allocation); next_block
/// converts them straight into the engine's pinned fp32 staging.
class ChunkStreamSource final : public SampleSource {
 public:
  ChunkStreamSource(std::istream& in, Index rows, std::size_t buffer_frames, std::uint64_t seed)
      : in_(&in), rows_(rows), buffer_(std::max<std::size_t>(1, buffer_frames)), seed_(seed) {
    if (rows < 1) throw ShapeMismatch("ChunkStreamSource: rows must be >= 1");
  }
  std::optional<Sample> next() override {
    if (pos_ == order_.size() && !refill()) return std::nullopt;
    const double* src = block_.data() + order_[pos_++] * std::size_t(rows_);
    Vector v(rows_);
    std::memcpy(v.data(), src, std::size_t(rows_) * sizeof(double));
    return Sample{std::move(v), t_++};
  }
  std::size_t next_block(std::size_t n, Index F, float* dst, std::uint64_t* index) override {
    if (F != rows_) throw ShapeMismatch("online_step: frame size vs dictionary rows");
    std::size_t m = 0;
    while (m < n) {
      if (pos_ == order_.size() && !refill()) break;
      const std::size_t take = std::min(n - m, order_.size() - pos_);
      for (std::size_t i = 0; i < take; ++i) {
        const double* src = block_.data() + order_[pos_ + i] * std::size_t(F);
        float* out = dst + (m + i) * std::size_t(F);
        for (Index f = 0; f < F; ++f) out[f] = float(src[f]);
        index[m + i] = t_++;
      }
      pos_ += take;
      m += take;
    }
    return m;
  }
  void seek(std::uint64_t) override { throw IoError("ChunkStreamSource: stream input is not seekable"); }
  std::optional<std::uint64_t> size() const override { return std::nullopt; }

 private:
  std::size_t pending_frames() const { return pending_.size() / std::size_t(rows_); }
  // one chunk appended to pending_ (false at a clean end of stream)
  bool read_chunk() {
    unsigned char head[8];
    in_->read(reinterpret_cast<char*>(head), 8);
    if (in_->gcount() == 0) return false;
    if (in_->gcount() != 8) throw TruncatedPayload("stream chunk header truncated");
    std::uint64_t count = 0;
    for (int i = 7; i >= 0; --i) count = (count << 8) | head[i];
    const std::size_t F = std::size_t(rows_);
    constexpr std::uint64_t kPiece = 4096;  // frames decoded per read
    std::vector<unsigned char> raw;
    for (std::uint64_t done = 0; done < count;) {
      const std::size_t nf = std::size_t(std::min(kPiece, count - done));
      raw.resize(nf * F * 8);
      in_->read(reinterpret_cast<char*>(raw.data()), std::streamsize(raw.size()));
      if (in_->gcount() != std::streamsize(raw.size())) throw TruncatedPayload("stream frame truncated");
      const std::size_t base = pending_.size();
      pending_.resize(base + nf * F);
      for (std::size_t i = 0; i < nf * F; ++i) {
        std::uint64_t bits = 0;
        for (int b = 7; b >= 0; --b) bits = (bits << 8) | raw[8 * i + std::size_t(b)];
        double x;
        std::memcpy(&x, &bits, 8);
        if (!std::isfinite(x) || x < 0.0) throw NonFiniteEntry("stream frame with invalid entries");
        pending_[base + i] = x;
      }
      done += nf;
    }
    return true;
  }
  bool refill() {
    while (pending_frames() < buffer_ && read_chunk()) {
    }
    if (pending_.empty()) return false;
    const std::size_t len = std::min(buffer_, pending_frames());
    const std::size_t F = std::size_t(rows_);
    block_.assign(pending_.begin(), pending_.begin() + std::ptrdiff_t(len * F));
    pending_.erase(pending_.begin(), pending_.begin() + std::ptrdiff_t(len * F));
    order_ = detail::shuffled_range(len, seed_, blocks_++);
    pos_ = 0;
    return true;
  }
  std::istream* in_;
  Index rows_;
  std::size_t buffer_;
  std::uint64_t seed_;
  std::uint64_t t_ = 0;
  std::uint64_t blocks_ = 0;
  std::vector<double> pending_;  // frames read ahead, arrival order
  std::vector<double> block_;    // the current buffer
  std::vector<std::uint64_t> order_;
  std::size_t pos_ = 0;
};

namespace detail {

/// RAII owner of one device engine plus pinned staging for frame blocks.
class OnlineEngine {
 public:
  OnlineEngine(Index F, Index K, int beta, int iters, double eps, RestartMode mode, std::uint64_t seed,
               std::int64_t n_store)
      : F_(F), K_(K), beta_(beta), iters_(iters), eps_(eps), mode_(mode), seed_(seed), n_store_(n_store) {
    isnmf_online_config c{};
    c.F = F;
    c.K = K;
    c.beta = beta;
    c.inner_iters = iters;
    c.epsilon = eps;
    c.restart = mode == RestartMode::warm ? ISNMF_RESTART_WARM : ISNMF_RESTART_FRESH;
    c.seed = seed;
    c.n_store = n_store;
    check(isnmf_online_create(&ctx_, &c));
  }
  ~OnlineEngine() {
    if (ctx_) isnmf_online_destroy(ctx_);
    if (stage_) isnmf_host_free(stage_);
  }
  OnlineEngine(const OnlineEngine&) = delete;
  OnlineEngine& operator=(const OnlineEngine&) = delete;
  bool matches(Index F, Index K, int beta, int iters, double eps, RestartMode mode, std::uint64_t seed,
               std::int64_t n_store) const {
    return F == F_ && K == K_ && beta == beta_ && iters == iters_ && eps == eps_ && mode == mode_ && seed == seed_ &&
           n_store == n_store_;
  }
  isnmf_online* ctx() { return ctx_; }
  float* staging(std::size_t frames) {
    if (frames > stage_frames_) {
      if (stage_) isnmf_host_free(stage_);
      stage_ = static_cast<float*>(isnmf_host_alloc(std::int64_t(frames * size_t(F_) * sizeof(float))));
      if (!stage_) check(ISNMF_E_CUDA);
      stage_frames_ = frames;
      index_.resize(frames);
    }
    return stage_;
  }
  std::uint64_t* index() { return index_.data(); }
  std::uint64_t warm_hash = 0;

 private:
  isnmf_online* ctx_ = nullptr;
  Index F_, K_;
  int beta_, iters_;
  double eps_;
  RestartMode mode_;
  std::uint64_t seed_;
  std::int64_t n_store_;
  float* stage_ = nullptr;
  std::size_t stage_frames_ = 0;
  std::vector<std::uint64_t> index_;
};

inline std::uint64_t hash_matrix(const Matrix& m) {  // FNV-1a over the bytes
  std::uint64_t h = 1469598103934665603ULL;
  const auto* p = reinterpret_cast<const unsigned char*>(m.data());
  const size_t n = size_t(m.size()) * sizeof(double);
  for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 1099511628211ULL;
  return h ^ std::uint64_t(m.rows()) ^ (std::uint64_t(m.cols()) << 32);
}

}  // namespace detail

/// Streaming trainer state (online.hpp:224-248).  `engine` is the device
/// context the fields are mirrored into during a call; copies share it, and
/// every call re-pushes the copy's own fields first.
struct OnlineState {
  Dictionary dict;
  std::uint64_t t = 0;
  Matrix pending_a;
  Matrix pending_b;
  Matrix warm_h;  // K x N in warm mode, empty in fresh mode
  double rho = 1.0;
  RestartMode restart = RestartMode::fresh;
  std::uint64_t seed = 0;
  double last_delta = std::numeric_limits<double>::infinity();
  std::uint64_t commits = 0;
  TrainReport trace;
  double pending_div = 0.0;
  std::uint64_t pending_count = 0;
  double last_minibatch_obj = 0.0;
  std::shared_ptr<detail::OnlineEngine> engine;

  Index rows() const { return dict.w.rows(); }
  Index atoms() const { return dict.w.cols(); }
};

namespace detail {

inline OnlineEngine& bind_engine(OnlineState& st, const SolverConfig& cfg) {
  const std::int64_t n_store = st.restart == RestartMode::warm ? std::int64_t(st.warm_h.cols()) : 0;
  const int iters = cfg.effective_inner_iters();
  if (!st.engine || !st.engine->matches(st.rows(), st.atoms(), cfg.beta, iters, cfg.epsilon, st.restart, st.seed,
                                        n_store))
    st.engine = std::make_shared<OnlineEngine>(st.rows(), st.atoms(), cfg.beta, iters, cfg.epsilon, st.restart,
                                               st.seed, n_store);
  return *st.engine;
}

/// Host fields -> device (the warm store only when its bytes changed).
inline void push(OnlineState& st, OnlineEngine& e) {
  isnmf_online* c = e.ctx();
  check(isnmf_online_set_dictionary(c, st.dict.w.data(), st.dict.a.data(), st.dict.b.data()));
  check(isnmf_online_set_pending(c, st.pending_a.data(), st.pending_b.data(), st.pending_div, st.pending_count));
  check(isnmf_online_set_counters(c, st.t, st.commits, st.rho));
  if (st.restart == RestartMode::warm) {
    const std::uint64_t h = hash_matrix(st.warm_h);
    if (h != e.warm_hash) {
      check(isnmf_online_set_warm_h(c, st.warm_h.data()));
      e.warm_hash = h;
    }
  }
}

/// Device -> host fields.
inline void pull(OnlineState& st, OnlineEngine& e, bool with_warm = true) {
  isnmf_online* c = e.ctx();
  check(isnmf_online_get_dictionary(c, st.dict.w.data(), st.dict.a.data(), st.dict.b.data()));
  check(isnmf_online_get_pending(c, st.pending_a.data(), st.pending_b.data(), &st.pending_div, &st.pending_count));
  double rho = 0.0;
  check(isnmf_online_get_counters(c, &st.t, &st.commits, &rho, &st.last_delta, &st.last_minibatch_obj));
  if (with_warm && st.restart == RestartMode::warm) {
    check(isnmf_online_get_warm_h(c, st.warm_h.data()));
    e.warm_hash = hash_matrix(st.warm_h);
  }
}

}  // namespace detail

/// Initial state from an l1-normalised nonnegative W0 (online.hpp:254-288).
inline OnlineState make_online_state(const Matrix& w0, const SolverConfig& config,
                                     std::optional<std::uint64_t> dataset_size, const Matrix* dataset = nullptr) {
  config.validate();
  if (w0.anyNegative() || !w0.allFinite()) throw NonPositiveInit("online: W0 must be nonnegative and finite");
  for (Index k = 0; k < w0.cols(); ++k) {
    double s = 0.0;
    for (Index f = 0; f < w0.rows(); ++f) s += w0(f, k);
    if (!(s > 0.0)) throw ZeroColumn("online: W0 has an all-zero column");
    if (std::abs(s - 1.0) > 1e-8) throw NonPositiveInit("online: W0 columns must be l1-normalized");
  }
  OnlineState st;
  st.dict.w = w0;
  st.dict.a = Matrix(w0.rows(), w0.cols());
  for (Index i = 0; i < w0.size(); ++i) st.dict.a.data()[i] = config.init_stats_weight * w0.data()[i] * w0.data()[i];
  st.dict.b = Matrix::Constant(w0.rows(), w0.cols(), config.init_stats_weight);
  st.pending_a = Matrix::Zero(w0.rows(), w0.cols());
  st.pending_b = Matrix::Zero(w0.rows(), w0.cols());
  st.restart = config.restart;
  st.seed = config.seed;
  st.rho = dataset_size ? std::pow(config.r, double(config.beta) / double(*dataset_size)) : 1.0;
  if (config.restart == RestartMode::warm) {
    if (!dataset) throw EmptyDataset("online: warm restarts need an in-memory dataset");
    st.warm_h = default_h0(*dataset, w0, config.epsilon);
  }
  st.trace.stage = "online";
  st.trace.config = config;
  st.trace.seed = config.seed;
  return st;
}

/// dictionary_commit (online.hpp:318-337) on the device.
inline void dictionary_commit(OnlineState& state) {
  SolverConfig cfg = state.trace.config;
  cfg.restart = state.restart;
  detail::OnlineEngine& e = detail::bind_engine(state, cfg);
  detail::push(state, e);
  detail::check(isnmf_online_commit(e.ctx()));
  detail::pull(state, e);
}

/// One sample through the engine (online.hpp:342-368): solve, statistics,
/// commit every beta samples.  A device round trip per call — drive long
/// streams through online_resume, which batches frames.
inline void online_step(OnlineState& state, const Sample& sample, const SolverConfig& config) {
  if (sample.frame.size() != state.rows()) throw ShapeMismatch("online_step: frame size vs dictionary rows");
  detail::OnlineEngine& e = detail::bind_engine(state, config);
  detail::push(state, e);
  std::vector<float> f(size_t(sample.frame.size()));
  for (Index i = 0; i < sample.frame.size(); ++i) f[size_t(i)] = float(sample.frame[i]);
  const std::uint64_t idx = sample.index;
  std::int32_t stopped = 0;
  detail::check(isnmf_online_run(e.ctx(), f.data(), state.rows(), 1, state.restart == RestartMode::warm ? &idx : nullptr,
                                 ~std::uint64_t(0), 0.0, &stopped));
  detail::pull(state, e);
}

/// Invoked after every dictionary commit (timer paused); return false to stop.
using OnlineCallback = std::function<bool(OnlineState&)>;

/// Continues training from a state (online.hpp:375-407).
inline void online_resume(OnlineState& state, SampleSource& source, const SolverConfig& config,
                          const OnlineCallback& callback = {}, const Clock& clock = steady_clock_seconds()) {
  config.validate();
  const std::uint64_t budget = config.max_epochs_or_samples;
  const double eta = config.effective_eta(state.rows(), state.atoms());
  if (state.t > 0 && state.t < budget) source.seek(state.t);
  detail::OnlineEngine& e = detail::bind_engine(state, config);
  detail::push(state, e);
  const std::uint64_t beta = std::uint64_t(config.beta);
  // look ahead several mini-batches only when nothing can stop the run at a
  // commit (exact source positioning otherwise)
  const bool batched = !callback && !(eta > 0.0);
  const std::uint64_t chunk = batched ? 64 * beta : beta;
  const Index F = state.rows();
  detail::PausableTimer timer(clock);
  bool stop = false;
  while (!stop && state.t < budget) {
    const std::uint64_t to_commit = beta - state.t % beta;
    std::uint64_t want = to_commit + (chunk > beta ? chunk - beta : 0);
    want = std::min<std::uint64_t>(want, budget - state.t);
    float* stage = e.staging(size_t(want));
    const std::size_t n = source.next_block(size_t(want), F, stage, e.index());
    if (n == 0) break;
    timer.pause();  // read the elapsed training time so far (pause + resume is a no-op)
    const double t_run = timer.elapsed();
    timer.resume();
    detail::check(isnmf_online_clear_trace(e.ctx()));
    std::int32_t stopped = 0;
    detail::check(isnmf_online_run(e.ctx(), stage, F, std::int64_t(n),
                                   state.restart == RestartMode::warm ? e.index() : nullptr, ~std::uint64_t(0), eta,
                                   &stopped));
    const bool committed = (state.t % beta) + n >= beta;
    std::vector<std::uint64_t> ts(n / beta + 2);
    std::vector<double> objs(ts.size()), secs(ts.size());
    std::int64_t np = 0;
    detail::check(isnmf_online_get_trace(e.ctx(), ts.data(), objs.data(), secs.data(), std::int64_t(ts.size()), &np));
    if (callback && committed) {
      detail::pull(state, e);
      timer.pause();
      for (std::int64_t i = 0; i < np; ++i) state.trace.points.push_back({ts[size_t(i)], timer.elapsed(), objs[size_t(i)], std::nullopt});
      if (!callback(state)) stop = true;
      timer.resume();
      if (eta > 0.0 && state.last_delta < eta) stop = true;
      if (!stop) detail::push(state, e);
    } else {
      std::uint64_t t_dev = 0, commits = 0;
      double rho = 0.0;
      detail::check(isnmf_online_get_counters(e.ctx(), &t_dev, &commits, &rho, &state.last_delta,
                                              &state.last_minibatch_obj));
      state.t = t_dev;
      state.commits = commits;
      for (std::int64_t i = 0; i < np; ++i)
        state.trace.points.push_back({ts[size_t(i)], t_run + secs[size_t(i)], objs[size_t(i)], std::nullopt});
      if (stopped) stop = true;
      if (eta > 0.0 && committed && state.last_delta < eta) stop = true;
    }
    if (n < want) break;  // source exhausted
  }
  timer.pause();
  detail::pull(state, e);
  if (state.trace.points.empty() && state.pending_count > 0)
    state.trace.points.push_back(
        {state.t, timer.elapsed(), state.pending_div / double(state.pending_count), std::nullopt});
  if (!state.trace.points.empty()) state.trace.final_train_obj = state.trace.points.back().train_obj;
}

/// Runs the streaming trainer over a source (online.hpp:413-419).
inline OnlineState online_train(SampleSource& source, const SolverConfig& config, const Matrix& w0,
                                const OnlineCallback& callback = {}, const Clock& clock = steady_clock_seconds()) {
  OnlineState state = make_online_state(w0, config, source.size(), source.dataset());
  online_resume(state, source, config, callback, clock);
  return state;
}

// --- checkpoints (online.hpp:421-489) ------------------------------------
// "ISCK" | u32 version | u32 restart (0 warm, 1 fresh) | u64 t | u64 seed |
// u64 commits | f64 rho (as u64 bits) | matrices W, A, B, pending_a,
// pending_b [, warm_h in warm mode].  The host fields are the state of record
// (online_resume pulls them from the device before returning), and the
// per-sample randomness is a function of (seed, t), so a fresh-mode run
// resumed from a checkpoint reproduces the uninterrupted one bit-exactly.

inline constexpr char kCheckpointMagic[4] = {'I', 'S', 'C', 'K'};
inline constexpr std::uint32_t kCheckpointFormatVersion = 1;

inline void save_checkpoint(std::ostream& out, const OnlineState& st) {
  detail::put_raw(out, kCheckpointMagic, 4);
  detail::put_le<std::uint32_t>(out, kCheckpointFormatVersion);
  detail::put_le<std::uint32_t>(out, st.restart == RestartMode::warm ? 0u : 1u);
  detail::put_le<std::uint64_t>(out, st.t);
  detail::put_le<std::uint64_t>(out, st.seed);
  detail::put_le<std::uint64_t>(out, st.commits);
  std::uint64_t rho_bits;
  std::memcpy(&rho_bits, &st.rho, 8);
  detail::put_le<std::uint64_t>(out, rho_bits);
  save_matrix(out, st.dict.w);
  save_matrix(out, st.dict.a);
  save_matrix(out, st.dict.b);
  save_matrix(out, st.pending_a);
  save_matrix(out, st.pending_b);
  if (st.restart == RestartMode::warm) save_matrix(out, st.warm_h);
}

inline void save_checkpoint(const std::string& path, const OnlineState& st) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("cannot open for writing: " + path);
  save_checkpoint(out, st);
  out.flush();
  if (!out) throw IoError("write failed: " + path);
}

inline OnlineState load_checkpoint(std::istream& in) {
  char magic[4];
  detail::get_raw(in, magic, 4, "checkpoint magic");
  if (std::memcmp(magic, kCheckpointMagic, 4) != 0) throw BadMagic("not a checkpoint file");
  const auto version = detail::get_le<std::uint32_t>(in, "checkpoint version");
  if (version != kCheckpointFormatVersion) throw BadMagic("unsupported checkpoint version " + std::to_string(version));
  const auto restart = detail::get_le<std::uint32_t>(in, "restart mode");
  if (restart > 1) throw UnsupportedFormat("invalid restart mode in checkpoint");
  OnlineState st;
  st.restart = restart == 0 ? RestartMode::warm : RestartMode::fresh;
  st.t = detail::get_le<std::uint64_t>(in, "t");
  st.seed = detail::get_le<std::uint64_t>(in, "seed");
  st.commits = detail::get_le<std::uint64_t>(in, "commits");
  const auto rho_bits = detail::get_le<std::uint64_t>(in, "rho");
  std::memcpy(&st.rho, &rho_bits, 8);
  st.dict.w = load_matrix(in);
  st.dict.a = load_matrix(in);
  st.dict.b = load_matrix(in);
  st.pending_a = load_matrix(in);
  st.pending_b = load_matrix(in);
  if (st.restart == RestartMode::warm) st.warm_h = load_matrix(in);
  st.trace.stage = "online";
  st.trace.seed = st.seed;
  return st;
}

inline OnlineState load_checkpoint(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open: " + path);
  return load_checkpoint(in);
}

}  // namespace isnmf
