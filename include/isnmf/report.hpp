// isnmf-b200 C++ API — run traces (reference proj/include/isnmf/report.hpp:18-34).
// Only the structs that trainer states carry; the CSV / JSON exporters of the
// reference (report.hpp:46-157) are persistence, outside this engine's scope.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "model.hpp"

namespace isnmf {

/// One trace row: samples seen (online) or epoch (batch), training wall-clock
/// excluding callbacks, the training objective and an optional held-out value.
struct TracePoint {
  std::uint64_t samples = 0;
  double seconds = 0.0;
  double train_obj = 0.0;
  std::optional<double> heldout;
};

/// The record of one training run.
struct TrainReport {
  std::string stage;  // "batch" or "online"
  SolverConfig config;
  std::uint64_t seed = 0;
  std::string final_w_path;
  double final_train_obj = 0.0;
  std::vector<TracePoint> points;
};

}  // namespace isnmf
