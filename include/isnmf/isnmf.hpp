// isnmf-b200 C++ API — umbrella header of the hot-path subset of the
// reference's proj/include/isnmf/isnmf.hpp plus the §8(f) rows built so far:
// held-out evaluation, matrix files, checkpoints and the spectrogram front end.
// WAV decoding, the experiment grid and report export are not part of this
// engine.
#pragma once

#include "batch.hpp"
#include "errors.hpp"
#include "harness.hpp"
#include "io.hpp"
#include "kernels.hpp"
#include "matrix.hpp"
#include "model.hpp"
#include "online.hpp"
#include "report.hpp"
#include "rng.hpp"
#include "spectrogram.hpp"
