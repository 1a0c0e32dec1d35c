// isnmf-b200 C++ API — the seeded random streams of the reference
// (proj/include/isnmf/rng.hpp:10-44), re-expressed: splitmix64 finaliser,
// stream mixing, std::mt19937_64 engines, 53-bit uniforms and rejection-sampled
// integers.  Results are bit-identical to the reference's; the device
// fresh-restart kernel (K0 in paper_1106_4198_b200/csrc/kernels.cuh) reproduces
// make_engine(mix_seed(seed, t)) as well.
#pragma once

#include <cstdint>
#include <random>

namespace isnmf {

namespace detail {
constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
constexpr std::uint64_t kMix1 = 0xbf58476d1ce4e5b9ULL;
constexpr std::uint64_t kMix2 = 0x94d049bb133111ebULL;
constexpr std::uint64_t xorshift(std::uint64_t v, int s) { return v ^ (v >> s); }
}  // namespace detail

/// splitmix64 finaliser of x (Steele, Lea & Flood), used to derive streams.
inline std::uint64_t splitmix64(std::uint64_t x) {
  using namespace detail;
  return xorshift(xorshift(xorshift(x + kGolden, 30) * kMix1, 27) * kMix2, 31);
}

/// Independent stream id for (seed, stream): both are finalised, the stream complemented.
inline std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t stream) {
  const std::uint64_t a = splitmix64(seed), b = splitmix64(~stream);
  return splitmix64(a ^ b);
}

/// std::mt19937_64 seeded with splitmix64(seed).
inline std::mt19937_64 make_engine(std::uint64_t seed) { return std::mt19937_64{splitmix64(seed)}; }

/// [0, 1) from the top 53 bits of one draw (library-independent).
inline double uniform01(std::mt19937_64& rng) {
  constexpr double kScale = 1.0 / 9007199254740992.0;  // 2^-53
  return double(rng() >> 11) * kScale;
}

/// (0, 1] as the complement of uniform01.
inline double uniform_open01(std::mt19937_64& rng) { return 1.0 - uniform01(rng); }

/// [0, n) without modulo bias: draws at or above the largest multiple of n are rejected.
inline std::uint64_t uniform_below(std::mt19937_64& rng, std::uint64_t n) {
  constexpr std::uint64_t kMax = ~std::uint64_t{0};
  const std::uint64_t cut = kMax - kMax % n;
  for (;;) {
    const std::uint64_t x = rng();
    if (x < cut) return x % n;
  }
}

}  // namespace isnmf
