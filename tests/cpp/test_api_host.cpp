// Host-side parts of the C++ API (no device needed): the reference's
// test_core.cpp cases that do not touch the engine, plus sources and helpers.
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

TEST_CASE("frobenius_delta basics (test_core.cpp:32-45)") {
  Matrix a = random_positive(4, 3, 1);
  CHECK(frobenius_delta(a, a) == 0.0);
  Matrix b = a;
  b(2, 1) += 3.0;
  CHECK(std::abs(frobenius_delta(b, a) - 3.0) < 1e-15);
  CHECK(std::abs(frobenius_delta(Matrix::Ones(2, 2), Matrix::Zero(2, 2)) - 2.0) < 1e-15);
  CHECK_THROWS_AS(frobenius_delta(a, Matrix::Zero(3, 3)), ShapeMismatch);
}

TEST_CASE("solver config validation (test_core.cpp:162-181)") {
  SolverConfig c;
  CHECK_NOTHROW(c.validate());
  c.k = 0;
  CHECK_THROWS_AS(c.validate(), NegativeInput);
  c = SolverConfig{};
  c.epsilon = 0.0;
  CHECK_THROWS_AS(c.validate(), NegativeInput);
  c = SolverConfig{};
  c.r = 1.5;
  CHECK_THROWS_AS(c.validate(), NegativeInput);
  c = SolverConfig{};
  CHECK(c.effective_inner_iters() == 1);
  c.restart = RestartMode::fresh;
  CHECK(c.effective_inner_iters() == 100);
  c.inner_iters = 7;
  CHECK(c.effective_inner_iters() == 7);
  CHECK_REL(SolverConfig{}.effective_eta(25, 4), 1e-6 * 10.0, 1e-12);
  CHECK(restart_mode_from_string("fresh") == RestartMode::fresh);
  CHECK_THROWS_AS(restart_mode_from_string("lukewarm"), UnsupportedFormat);
}

TEST_CASE("rng streams are deterministic and uniform_below is in range") {
  auto a = make_engine(mix_seed(3, 9)), b = make_engine(mix_seed(3, 9));
  for (int i = 0; i < 100; ++i) CHECK(a() == b());
  auto c = make_engine(5);
  for (int i = 0; i < 1000; ++i) {
    const double u = uniform01(c);
    CHECK(u >= 0.0 && u < 1.0);
    CHECK(uniform_below(c, 7) < 7);
  }
  CHECK(splitmix64(0) == 0xe220a8397b1dcdafULL);  // splitmix64 published first output for state 0
}

TEST_CASE("cycling source: every frame once per cycle, exact seek (online.hpp:53-94)") {
  Matrix v = random_positive(3, 10, 4);
  CyclingSource s(v, 11);
  std::vector<int> seen(10, 0);
  std::vector<std::uint64_t> first;
  for (int i = 0; i < 10; ++i) {
    auto x = s.next();
    REQUIRE(x.has_value());
    seen[size_t(x->index)]++;
    first.push_back(x->index);
    CHECK(x->frame[0] == v(0, Index(x->index)));
  }
  for (int k : seen) CHECK(k == 1);
  CyclingSource t(v, 11);
  t.seek(7);
  CHECK(t.next()->index == first[7]);
  float buf[3 * 4];
  std::uint64_t idx[4];
  CyclingSource u(v, 11);
  CHECK(u.next_block(4, 3, buf, idx) == 4);
  for (int i = 0; i < 4; ++i) CHECK(idx[i] == first[size_t(i)]);
  CHECK(*s.size() == 10 && s.dataset() == &v);
}

TEST_CASE("generator and chunk-stream sources (online.hpp:98-220)") {
  GeneratorSource g([](std::uint64_t i) { return Vector::Constant(2, double(i)); }, 5, 2, 3);
  std::vector<int> seen(5, 0);
  for (int i = 0; i < 5; ++i) seen[size_t(g.next()->index)]++;
  CHECK(!g.next().has_value());
  for (int k : seen) CHECK(k == 1);
  std::string bytes;
  auto put64 = [&](std::uint64_t x) {
    for (int i = 0; i < 8; ++i) bytes.push_back(char((x >> (8 * i)) & 0xff));
  };
  put64(2);
  for (double d : {1.0, 2.0, 3.0, 4.0}) {
    std::uint64_t b;
    std::memcpy(&b, &d, 8);
    put64(b);
  }
  std::istringstream in(bytes);
  ChunkStreamSource cs(in, 2, 4, 1);
  double tot = 0.0;
  int n = 0;
  while (auto x = cs.next()) {
    tot += x->frame.sum();
    ++n;
  }
  CHECK(n == 2 && tot == 10.0);
  std::istringstream bad(bytes.substr(0, 12));
  ChunkStreamSource cb(bad, 2, 4, 1);
  CHECK_THROWS_AS(cb.next(), TruncatedPayload);
  CHECK_THROWS_AS(cs.seek(0), IoError);
}

TEST_CASE("make_online_state validates W0 and sets A0, B0, rho (online.hpp:254-288)") {
  SolverConfig c;
  c.k = 2;
  c.beta = 5;
  c.r = 0.49;
  c.restart = RestartMode::fresh;
  Matrix w = Matrix::Constant(4, 2, 0.25);
  OnlineState st = make_online_state(w, c, 10);
  CHECK(std::abs(st.rho - 0.7) < 1e-15);
  CHECK(st.dict.a(1, 1) == 0.0625 && st.dict.b(0, 0) == 1.0);
  CHECK(make_online_state(w, c, std::nullopt).rho == 1.0);
  CHECK_THROWS_AS(make_online_state(Matrix::Constant(4, 2, 1.0), c, 10), NonPositiveInit);
  c.restart = RestartMode::warm;
  CHECK_THROWS_AS(make_online_state(w, c, 10), EmptyDataset);
  Matrix v = random_positive(4, 6, 2);
  OnlineState sw = make_online_state(w, c, 6, &v);
  CHECK(sw.warm_h.rows() == 2 && sw.warm_h.cols() == 6);
  CHECK_REL(sw.warm_h(1, 3), v.mean() / (2 * 0.25), 1e-14);
}

TEST_CASE("init_from_samples / default_h0 (batch.hpp:58-78)") {
  Matrix v = random_positive(5, 9, 3);
  Matrix w1 = init_from_samples(v, 3, 7), w2 = init_from_samples(v, 3, 7);
  CHECK(frobenius_delta(w1, w2) == 0.0);
  for (Index k = 0; k < 3; ++k) {
    double s = 0.0;
    for (Index f = 0; f < 5; ++f) s += w1(f, k);
    CHECK(std::abs(s - 1.0) < 1e-12);
  }
  CHECK_THROWS_AS(init_from_samples(Matrix(5, 0), 3, 1), EmptyDataset);
}

MT_MAIN()

TEST_CASE("matrix files round-trip bit-exactly and reject bad input (io.hpp)") {
  Matrix m = random_positive(7, 5, 11);
  m(3, 2) = 0.0;
  m(0, 0) = 1e-300;
  std::stringstream ss;
  save_matrix(ss, m);
  CHECK(ss.str().size() == 4 + 4 + 16 + 8 * 35);
  Matrix r = load_matrix(ss);
  CHECK(r.rows() == 7 && r.cols() == 5);
  CHECK(std::memcmp(r.data(), m.data(), 35 * sizeof(double)) == 0);
  std::stringstream bad("ISNX0000");
  CHECK_THROWS_AS(load_matrix(bad), BadMagic);
  std::string s = ss.str();
  std::stringstream trunc(s.substr(0, s.size() - 3));
  CHECK_THROWS_AS(load_matrix(trunc), TruncatedPayload);
  Matrix neg = m;
  neg(1, 1) = -1.0;
  std::stringstream sn;
  save_matrix(sn, neg);
  CHECK_THROWS_AS(load_matrix(sn), NegativeEntry);
}

TEST_CASE("checkpoints round-trip every field bit-exactly (online.hpp:421-489)") {
  for (RestartMode mode : {RestartMode::warm, RestartMode::fresh}) {
    OnlineState st;
    st.dict.w = random_positive(9, 3, 1);
    st.dict.a = random_positive(9, 3, 2);
    st.dict.b = random_positive(9, 3, 3);
    st.pending_a = random_positive(9, 3, 4);
    st.pending_b = random_positive(9, 3, 5);
    if (mode == RestartMode::warm) st.warm_h = random_positive(3, 11, 6);
    st.restart = mode;
    st.t = 123456789012ULL;
    st.seed = 0xdeadbeefULL;
    st.commits = 77;
    st.rho = 0.95967;
    std::stringstream ss;
    save_checkpoint(ss, st);
    OnlineState r = load_checkpoint(ss);
    CHECK(r.restart == mode && r.t == st.t && r.seed == st.seed && r.commits == st.commits);
    CHECK(std::memcmp(&r.rho, &st.rho, 8) == 0);
    const Matrix* a[] = {&st.dict.w, &st.dict.a, &st.dict.b, &st.pending_a, &st.pending_b, &st.warm_h};
    const Matrix* b[] = {&r.dict.w, &r.dict.a, &r.dict.b, &r.pending_a, &r.pending_b, &r.warm_h};
    for (int i = 0; i < 6; ++i) {
      CHECK(a[i]->rows() == b[i]->rows() && a[i]->cols() == b[i]->cols());
      CHECK(std::memcmp(a[i]->data(), b[i]->data(), size_t(a[i]->size()) * sizeof(double)) == 0);
    }
  }
  std::stringstream bad("ISCX");
  CHECK_THROWS_AS(load_checkpoint(bad), BadMagic);
  std::stringstream mode;
  mode.write("ISCK", 4);
  const unsigned char v1[4] = {1, 0, 0, 0}, m7[4] = {7, 0, 0, 0};
  mode.write(reinterpret_cast<const char*>(v1), 4);
  mode.write(reinterpret_cast<const char*>(m7), 4);
  CHECK_THROWS_AS(load_checkpoint(mode), UnsupportedFormat);
}

TEST_CASE("ChunkStreamSource: next() and the next_block fast path agree across chunks and buffers") {
  const Index F = 3;
  std::string bytes;
  auto put64 = [&](std::uint64_t v) {
    for (int i = 0; i < 8; ++i) bytes.push_back(char((v >> (8 * i)) & 0xff));
  };
  double val = 0.0;
  for (std::uint64_t count : {5u, 0u, 7u, 2u}) {  // 14 frames in ragged chunks (one empty)
    put64(count);
    for (std::uint64_t c = 0; c < count * std::uint64_t(F); ++c) {
      val += 1.0;
      std::uint64_t b;
      std::memcpy(&b, &val, 8);
      put64(b);
    }
  }
  std::istringstream in1(bytes), in2(bytes);
  ChunkStreamSource a(in1, F, 4, 9), b(in2, F, 4, 9);
  std::vector<double> seq;
  std::vector<std::uint64_t> idx;
  while (auto s = a.next()) {
    for (Index f = 0; f < F; ++f) seq.push_back(s->frame[f]);
    idx.push_back(s->index);
  }
  CHECK(seq.size() == 14 * 3);
  std::vector<float> blk(14 * 3);
  std::vector<std::uint64_t> bidx(14);
  std::size_t got = b.next_block(5, F, blk.data(), bidx.data());
  got += b.next_block(20, F, blk.data() + got * 3, bidx.data() + got);
  CHECK(got == 14);
  for (std::size_t i = 0; i < seq.size(); ++i) CHECK(blk[i] == float(seq[i]));
  for (std::size_t i = 0; i < 14; ++i) CHECK(bidx[i] == i && idx[i] == i);
  // within each 4-frame buffer the frames are the reference's permutation of arrival order
  for (std::size_t blk0 = 0; blk0 < 14; blk0 += 4) {
    const std::size_t len = std::min<std::size_t>(4, 14 - blk0);
    const auto perm = detail::shuffled_range(len, 9, blk0 / 4);
    for (std::size_t i = 0; i < len; ++i) CHECK(seq[(blk0 + i) * 3] == double(3 * (blk0 + perm[i]) + 1));
  }
  std::string bad = bytes;
  bad[8 + 8 * 4] = 0;
  bad[8 + 8 * 4 + 7] = char(0xff);  // frame 1, bin 1 becomes negative / non-finite
  std::istringstream in3(bad);
  ChunkStreamSource c(in3, F, 4, 9);
  CHECK_THROWS_AS(c.next(), NonFiniteEntry);
}
