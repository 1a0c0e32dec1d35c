// The reference's own unit tests (proj/tests/test_kernels.cpp, test_core.cpp
// rescale cases) restated against the isnmf-b200 C++ API, which computes on the
// B200 in fp32: tolerances that the reference states for fp64 are widened to
// the fp32 level and marked; plus trainer-level checks of online_train /
// online_resume / batch_train through the same API.
#include <sstream>

#include "isnmf/isnmf.hpp"


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


int main() {
  const Index F = 33, K = 3, N = 40;
  Matrix v = spectrogram(F, K, N, 41);
  Matrix w = normalized(random_positive(F, K, 42, 0.1, 1.0));
  for (int i = 0; i < 4; ++i) printf("%.17g\n", evaluate_heldout(w, v, 1e-12));
  for (int it : {1, 2, 5, 10, 20, 50}) printf("iters %d: %.17g\n", it, evaluate_heldout(w, v, 1e-12, it));
  return 0;
}
