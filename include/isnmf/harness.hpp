// Held-out evaluation (reference harness.hpp:17-37) on the device.  The rest
// of the reference harness (run_experiment, grid search, report export) is
// outside the engine's scope.
#pragma once

#include <cstdint>
#include <vector>

#include "errors.hpp"
#include "matrix.hpp"

namespace isnmf {

/// Refits activations of `test` from the reference's seed-deterministic
/// random init with `inner_iters` MM updates at frozen W and returns the mean
/// IS divergence per frame.  W is not modified.
inline double evaluate_heldout(const Matrix& w, const Matrix& test, double epsilon, int inner_iters = 100,
                               std::uint64_t seed = 0x45u) {
  if (w.rows() != test.rows()) throw ShapeMismatch("evaluate_heldout: W rows vs test rows");
  if (test.cols() == 0) throw EmptyDataset("evaluate_heldout: empty test set");
  std::vector<float> t32(std::size_t(test.size()));
  for (std::size_t i = 0; i < t32.size(); ++i) t32[i] = float(test.data()[i]);
  double out = 0.0;
  detail::check(isnmf_evaluate_heldout(t32.data(), test.rows(), test.rows(), test.cols(), w.data(), w.cols(), epsilon,
                                       inner_iters, seed, &out));
  return out;
}

}  // namespace isnmf
