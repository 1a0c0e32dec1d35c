"""GPU parity of the stateless kernels (kernels.hpp / model.hpp) through the C ABI.

Two layers: (1) the reference's own golden cases (proj/tests/test_kernels.cpp,
test_core.cpp) re-run on the device with fp32 tolerances, (2) seeded random
cases against the CPU fp64 oracle.  Tolerances (north_star): 1e-4 relative
for fp32-computed quantities; update_w / rescale / is_divergence run in fp64
on the device and are held to 1e-12.
"""
import math

import numpy as np
import pytest

import oracle as O
import paper_1106_4198_b200 as E
from oracle import random_positive

pytestmark = pytest.mark.gpu
RTOL = 1e-4


def rpv(n, seed, lo=0.05, hi=2.0):
    return random_positive(n, 1, seed, lo, hi)[:, 0].copy()


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


# ---- golden cases (test_kernels.cpp) on the device --------------------------------
def test_is_divergence_golden():
    y = rpv(16, 1)
    assert E.is_divergence(y, y, 1e-12) == 0.0
    expect = 2.0 * (0.5 + math.log(2.0) - 1.0)
    assert abs(E.is_divergence(np.ones(2), np.full(2, 2.0), 1e-15) - expect) <= 1e-9 * expect
    with pytest.raises(E.EngineError) as e:
        E.is_divergence(np.ones(3), np.ones(4), 1e-12)
    assert e.value.kind == "ShapeMismatch"
    neg = np.ones(3)
    neg[0] = -0.5
    with pytest.raises(E.EngineError) as e:
        E.is_divergence(neg, neg, 1e-12)
    assert e.value.kind == "NegativeInput"
    for trial in range(20):
        a, b = rpv(12, 300 + trial), rpv(12, 400 + trial)
        assert abs(E.is_divergence(a, b, 1e-12) - O.is_divergence(a, b, 1e-12)) <= 1e-12 * O.is_divergence(a, b, 1e-12)


def test_solve_h_golden():
    w = random_positive(6, 2, 11)
    h_star = rpv(2, 12)
    h = E.solve_h(w @ h_star, w, h_star, 25, 1e-14)
    assert rel(h, h_star) < 1e-5  # fp32 fixed point (reference: 1e-9 in fp64)
    h = E.solve_h(np.array([4.0]), np.array([[2.0]]), np.array([0.3]), 100, 1e-12)
    assert abs(h[0] - 2.0) <= 1e-6 * 2.0 * 4
    with pytest.raises(E.EngineError) as e:
        E.solve_h(rpv(3, 17), random_positive(3, 2, 16), np.zeros(2), 5, 1e-12)
    assert e.value.kind == "NonPositiveInit"


def test_solve_h_descends():
    w = random_positive(9, 3, 13)
    v = rpv(9, 14)
    h = rpv(3, 15)
    prev = O.is_divergence(v, w @ h, 1e-12)
    for _ in range(60):
        h = E.solve_h(v, w, h, 1, 1e-12)
        cur = O.is_divergence(v, w @ h, 1e-12)
        assert cur <= prev * (1 + 1e-6) + 1e-10
        prev = cur


def test_sample_stats_golden():
    a, b = E.batch_stats(np.array([[8.0]]), np.array([[2.0]]), np.array([[1.0]]), 1e-30)
    assert rel(a, 8.0) < 1e-6 and rel(b, 0.5) < 1e-6
    a, b = E.batch_stats(np.array([[0.0]]), np.array([[1.0]]), np.array([[1.0]]), 1.0)
    assert rel(a, 0.25) < 1e-6 and rel(b, 0.5) < 1e-6
    w = random_positive(7, 3, 21)
    h = random_positive(3, 1, 22)
    a, b = E.batch_stats(w @ h, w, h, 1e-30)
    assert rel(np.sqrt(a / b), w) < 1e-5


def test_update_w_golden():
    a = np.full((3, 2), 0.7)
    assert np.max(np.abs(E.update_w(a, a, np.full((3, 2), 0.123)) - 1.0)) < 1e-15
    assert abs(E.update_w(np.array([[4.0]]), np.array([[1.0]]), np.ones((1, 1)))[0, 0] - 2.0) <= 2e-15
    a, b = np.zeros((2, 1)), np.zeros((2, 1))
    a[0, 0], b[0, 0] = 1.0, 4.0
    w = E.update_w(a, b, np.array([[0.3], [0.7]]))
    assert abs(w[0, 0] - 0.5) < 1e-15 and w[1, 0] == 0.7
    with pytest.raises(E.EngineError) as e:
        E.update_w(np.ones((1, 1)), np.zeros((1, 1)), np.ones((1, 1)))
    assert e.value.kind == "InconsistentStats"


def test_rescale_golden():
    w, a, b, _ = E.rescale_dictionary(np.full((2, 1), 2.0), np.ones((2, 1)), np.ones((2, 1)))
    assert np.allclose(w, 0.5, rtol=1e-15) and np.allclose(a, 0.25, rtol=1e-15) and np.allclose(b, 4.0, rtol=1e-15)
    w0 = random_positive(6, 3, 2)
    h0 = random_positive(3, 5, 3)
    w2, _, _, h2 = E.rescale_dictionary(w0, random_positive(6, 3, 4), random_positive(6, 3, 5), h0)
    assert np.linalg.norm(w2 @ h2 - w0 @ h0) < 1e-12
    with pytest.raises(E.EngineError) as e:
        E.rescale_dictionary(np.zeros((3, 1)), np.zeros((3, 1)), np.zeros((3, 1)))
    assert e.value.kind == "ZeroColumn"


def test_objective_golden():
    w, h = random_positive(5, 2, 61), random_positive(2, 7, 62)
    assert E.objective(w @ h, w, h, 1e-30) < 1e-6  # fp32 reconstruction of an exact factorisation
    v, w, h = random_positive(6, 5, 63), random_positive(6, 2, 64), random_positive(2, 5, 65)
    assert rel(E.objective(v, w, h, 1e-12), O.objective(v, w, h, 1e-12)) < RTOL
    with pytest.raises(E.EngineError) as e:
        E.objective(np.zeros((6, 0)), w, np.zeros((2, 0)), 1e-12)
    assert e.value.kind == "EmptyDataset"


# ---- seeded random cases vs the oracle ----------------------------------------------
@pytest.mark.parametrize("F,K,N,iters", [(257, 10, 37, 5), (513, 20, 150, 10), (513, 50, 300, 10),
                                         (65, 3, 9, 100), (513, 64, 40, 3), (33, 1, 5, 7)])
def test_solve_h_matches_oracle(F, K, N, iters):
    from tools.synth import spectrogram_np, w_init
    v = spectrogram_np(F, K, N, seed=F + K).astype(np.float64)
    w = w_init(F, K, seed=K)
    h0 = np.ones((K, N))
    got = E.solve_h(v, w, h0, iters, 1e-12)
    ref = O.solve_h(v, w, h0, iters, 1e-12)
    assert rel(got, ref) < RTOL


@pytest.mark.parametrize("F,K,N", [(257, 10, 100), (513, 50, 4096), (100, 7, 3)])
def test_batch_stats_and_objective_match_oracle(F, K, N):
    from tools.synth import spectrogram_np, w_init
    v = spectrogram_np(F, K, N, seed=3).astype(np.float64)
    w = w_init(F, K, seed=4)
    h = np.random.default_rng(5).gamma(0.5, 1.0, size=(K, N)) + 1e-3
    a, b = E.batch_stats(v, w, h, 1e-12)
    ra, rb = O.batch_stats(v, w, h, 1e-12)
    assert rel(a, ra) < RTOL and rel(b, rb) < RTOL
    assert rel(E.objective(v, w, h, 1e-12), O.objective(v, w, h, 1e-12)) < RTOL
