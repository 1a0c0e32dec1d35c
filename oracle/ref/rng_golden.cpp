// TEST INFRASTRUCTURE ONLY (never linked into the engine): prints golden
// vectors of the reference's own random-number path, compiled straight from
// the reference header /root/reference/proj/include/isnmf/rng.hpp (the one
// reference source that builds without Eigen; oracle/Makefile target `ref`,
// output oracle/_ref/rng_golden).  tests/golden/gen_rng_golden.py turns the
// output into tests/golden/rng_streams.json.
//
// Streams: splitmix64 / mix_seed (rng.hpp:10-19); raw make_engine draws
// (rng.hpp:21-23); uniform01 / uniform_open01 (rng.hpp:27-34); uniform_below
// (rng.hpp:37-44); the fresh-restart draws make_engine(mix_seed(seed, t)) ->
// uniform_open01 x K (online.hpp:294-301); the CyclingSource Fisher-Yates order
// of one cycle (online.hpp:79-87, the swap loop driven by the reference's
// uniform_below); random_positive of the reference tests (test_kernels.cpp:13-19).
#include <cinttypes>
#include <cstdio>
#include <numeric>
#include <utility>
#include <vector>

#include "isnmf/rng.hpp"

using isnmf::make_engine;
using isnmf::mix_seed;

static void u64list(const char* name, const std::vector<std::uint64_t>& v, bool last = false) {
  std::printf("  \"%s\": [", name);
  for (std::size_t i = 0; i < v.size(); ++i) std::printf("%s\"%" PRIu64 "\"", i ? ", " : "", v[i]);
  std::printf("]%s\n", last ? "" : ",");
}
static void dlist(const char* name, const std::vector<double>& v, bool last = false) {
  std::printf("  \"%s\": [", name);
  for (std::size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? ", " : "", v[i]);
  std::printf("]%s\n", last ? "" : ",");
}

int main() {
  const std::vector<std::uint64_t> xs = {0, 1, 2, 42, 0x45, 0xE7A1, 1234567890123ULL, ~std::uint64_t(0)};
  std::printf("{\n");
  u64list("splitmix64_in", xs);
  std::vector<std::uint64_t> sm, ms;
  for (auto x : xs) sm.push_back(isnmf::splitmix64(x));
  u64list("splitmix64_out", sm);
  for (auto x : xs) ms.push_back(mix_seed(x, x * 3 + 1));  // mix_seed(x, 3x + 1)
  u64list("mix_seed_out", ms);
  {
    auto g = make_engine(7);
    std::vector<std::uint64_t> raw;
    for (int i = 0; i < 16; ++i) raw.push_back(g());
    u64list("engine7_raw16", raw);
  }
  {
    auto g = make_engine(11);
    std::vector<double> u;
    for (int i = 0; i < 16; ++i) u.push_back(isnmf::uniform01(g));
    dlist("engine11_uniform01", u);
    std::vector<double> o;
    for (int i = 0; i < 16; ++i) o.push_back(isnmf::uniform_open01(g));
    dlist("engine11_then_open01", o);
  }
  {
    auto g = make_engine(13);
    std::vector<std::uint64_t> b;
    const std::uint64_t ns[] = {1, 2, 3, 7, 100, 4097, 1ULL << 40, 0xFFFFFFFFFFFFFFF1ULL};
    for (int r = 0; r < 2; ++r)
      for (auto n : ns) b.push_back(isnmf::uniform_below(g, n));
    u64list("engine13_below", b);
  }
  {  // fresh_h_init draws (online.hpp:294-301): seed 1, t = 0, 1, 99, K = 5
    std::vector<double> f;
    for (std::uint64_t t : {0ULL, 1ULL, 99ULL}) {
      auto g = make_engine(mix_seed(1, t));
      for (int k = 0; k < 5; ++k) f.push_back(isnmf::uniform_open01(g));
    }
    dlist("fresh_seed1_t0_1_99_k5", f);
  }
  {  // CyclingSource cycle order (online.hpp:79-87): seed 5, cycles 0 and 1, N = 20
    std::vector<std::uint64_t> order;
    for (std::uint64_t cycle : {0ULL, 1ULL}) {
      std::vector<std::uint64_t> perm(20);
      std::iota(perm.begin(), perm.end(), std::uint64_t(0));
      auto g = make_engine(mix_seed(5, cycle));
      for (std::size_t i = perm.size(); i > 1; --i)
        std::swap(perm[i - 1], perm[static_cast<std::size_t>(isnmf::uniform_below(g, i))]);
      order.insert(order.end(), perm.begin(), perm.end());
    }
    u64list("cycling_seed5_n20_cycles01", order);
  }
  {  // random_positive(3, 2, seed 21, lo 0.05, hi 2.0) of the reference tests (column-major)
    auto g = make_engine(21);
    std::vector<double> m;
    for (int j = 0; j < 2; ++j)
      for (int i = 0; i < 3; ++i) m.push_back(0.05 + (2.0 - 0.05) * isnmf::uniform01(g));
    dlist("random_positive_3x2_seed21", m, true);
  }
  std::printf("}\n");
  return 0;
}
