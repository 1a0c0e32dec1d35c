"""Random streams pinned to the reference itself.

tests/golden/rng_streams.json was printed by the reference's own rng.hpp,
compiled here from /root/reference (tests/golden/gen_rng_golden.py).  Checked
against it: the CPU oracle's restatement (oracle/isnmf_oracle.hpp: splitmix64,
mix_seed, uniform01, the CyclingSource order, fresh_h_init, the tests'
random_positive) and the drop-in C++ header include/isnmf/rng.hpp (every
stream, via a small program compiled here).  The device mt19937_64 (K0,
fresh restarts) is held to the oracle by the fresh-restart GPU parity tests.
"""
import json
import os
import subprocess

import numpy as np

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = json.load(open(os.path.join(ROOT, "tests", "golden", "rng_streams.json")))


def u64(lst):
    return [int(x) for x in lst]


def test_oracle_splitmix_and_mix_seed():
    xs = u64(G["splitmix64_in"])
    assert [O.splitmix64(x) for x in xs] == u64(G["splitmix64_out"])
    assert [O.mix_seed(x, (3 * x + 1) % 2**64) for x in xs] == u64(G["mix_seed_out"])


def test_oracle_uniform01_and_random_positive():
    assert np.array_equal(O.uniform01(11, 16), np.array(G["engine11_uniform01"]))
    m = O.random_positive(3, 2, 21)
    assert np.array_equal(m.T.reshape(-1), np.array(G["random_positive_3x2_seed21"]))


def test_oracle_cycling_order():
    order = np.concatenate([O.cycle_permutation(5, c, 20) for c in (0, 1)]).astype(np.uint64)
    assert [int(x) for x in order] == u64(G["cycling_seed5_n20_cycles01"])


def test_oracle_fresh_h_init():
    # v = ones (mean 1), w = 1/K (K * mean(w) = 1): the scale is 1, h = the raw draws
    K, F = 5, 3
    v, w = np.ones(F), np.full((F, K), 1.0 / K)
    got = np.concatenate([O.fresh_h_init(v, w, 1e-12, 1, t) for t in (0, 1, 99)])
    assert np.allclose(got, G["fresh_seed1_t0_1_99_k5"], rtol=1e-15, atol=0)


PROGRAM = r"""
#include <cinttypes>
#include <cstdio>
#include <numeric>
#include <utility>
#include <vector>
#include "isnmf/rng.hpp"
using namespace isnmf;
int main() {
  const std::uint64_t xs[] = {0, 1, 2, 42, 0x45, 0xE7A1, 1234567890123ULL, ~std::uint64_t(0)};
  for (auto x : xs) std::printf("%" PRIu64 " %" PRIu64 "\n", splitmix64(x), mix_seed(x, x * 3 + 1));
  { auto g = make_engine(7); for (int i = 0; i < 16; ++i) std::printf("%" PRIu64 "\n", g()); }
  { auto g = make_engine(11); for (int i = 0; i < 16; ++i) std::printf("%.17g\n", uniform01(g));
    for (int i = 0; i < 16; ++i) std::printf("%.17g\n", uniform_open01(g)); }
  { auto g = make_engine(13); const std::uint64_t ns[] = {1, 2, 3, 7, 100, 4097, 1ULL << 40, 0xFFFFFFFFFFFFFFF1ULL};
    for (int r = 0; r < 2; ++r) for (auto n : ns) std::printf("%" PRIu64 "\n", uniform_below(g, n)); }
  for (std::uint64_t t : {0ULL, 1ULL, 99ULL}) { auto g = make_engine(mix_seed(1, t));
    for (int k = 0; k < 5; ++k) std::printf("%.17g\n", uniform_open01(g)); }
  return 0;
}
"""


def test_dropin_header_streams(tmp_path):
    src, exe = tmp_path / "rng.cpp", tmp_path / "rng"
    src.write_text(PROGRAM)
    subprocess.run(["g++", "-std=c++17", "-O1", f"-I{ROOT}/include", str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    it = iter(out)
    for sm, ms in zip(u64(G["splitmix64_out"]), u64(G["mix_seed_out"])):
        a, b = next(it).split()
        assert (int(a), int(b)) == (sm, ms)
    assert [int(next(it)) for _ in range(16)] == u64(G["engine7_raw16"])
    assert [float(next(it)) for _ in range(16)] == G["engine11_uniform01"]
    assert [float(next(it)) for _ in range(16)] == G["engine11_then_open01"]
    assert [int(next(it)) for _ in range(16)] == u64(G["engine13_below"])
    assert [float(next(it)) for _ in range(15)] == G["fresh_seed1_t0_1_99_k5"]
