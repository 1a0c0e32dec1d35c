// isnmf-b200 C++ API — umbrella header of the hot-path subset of the
// reference's proj/include/isnmf/isnmf.hpp (audio ingest, the experiment
// harness, matrix / checkpoint files and report export are not part of this
// engine).
#pragma once

#include "batch.hpp"
#include "errors.hpp"
#include "kernels.hpp"
#include "matrix.hpp"
#include "model.hpp"
#include "online.hpp"
#include "report.hpp"
#include "rng.hpp"
