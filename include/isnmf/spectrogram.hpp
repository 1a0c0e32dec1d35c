// Spectrogram front end (reference audio.hpp:121-187) on the device: the step
// that produces V.  WAV decoding and dataset files (audio.hpp:30-120, 189-206)
// stay outside the engine.
#pragma once

#include <cstdint>
#include <vector>

#include "errors.hpp"
#include "matrix.hpp"

namespace isnmf {

/// Power spectrogram with a sine analysis window: frame i covers samples
/// [i*hop, i*hop + window); F = window/2 + 1 bins, N = (len - window)/hop + 1
/// frames (fp64 FFT on the device; direct DFT for windows that are not powers of two).
inline Matrix stft_power(const std::vector<double>& samples, int window = 512, int hop = 256) {
  const std::int64_t frames =
      window >= 2 && hop >= 1 && samples.size() >= std::size_t(window) ? (std::int64_t(samples.size()) - window) / hop + 1
                                                                         : 0;
  Matrix power(Index(window >= 2 ? window / 2 + 1 : 1), Index(frames > 0 ? frames : 0));
  std::int64_t got = 0;
  detail::check(isnmf_stft_power(samples.data(), std::int64_t(samples.size()), window, hop, power.data(),
                                 std::int64_t(power.cols()), &got));
  return power;
}

struct FrameMeta {
  std::uint32_t file_index = 0;
  std::uint64_t frame_index = 0;
};

struct SpectrogramDataset {
  Matrix frames;
  double sample_rate = 0.0;
  std::vector<FrameMeta> meta;
  std::uint64_t discarded_count = 0;
};

/// Drops every frame whose total power sits more than |threshold_db| dB below the
/// loudest frame; retained frames keep their order (selection on the device).
inline SpectrogramDataset discard_silence(const Matrix& spec, double threshold_db = -60.0, double sample_rate = 0.0,
                                          const std::vector<FrameMeta>* meta = nullptr) {
  const Index n = spec.cols();
  if (meta && Index(meta->size()) != n) throw ShapeMismatch("discard_silence: metadata length vs frame count");
  std::vector<std::int64_t> keep(std::size_t(n > 0 ? n : 1));
  std::int64_t kept = 0;
  detail::check(isnmf_discard_silence(spec.data(), spec.rows(), n, threshold_db, keep.data(), &kept));
  SpectrogramDataset ds;
  ds.sample_rate = sample_rate;
  ds.discarded_count = std::uint64_t(n - kept);
  ds.frames = Matrix(spec.rows(), Index(kept));
  ds.meta.reserve(std::size_t(kept));
  for (std::int64_t j = 0; j < kept; ++j) {
    const Index src = Index(keep[std::size_t(j)]);
    for (Index f = 0; f < spec.rows(); ++f) ds.frames(f, Index(j)) = spec(f, src);
    ds.meta.push_back(meta ? (*meta)[std::size_t(src)] : FrameMeta{0, std::uint64_t(src)});
  }
  return ds;
}

}  // namespace isnmf
