"""Pins the CPU oracle to the reference's own golden values and properties.

Restates, case by case, /root/reference/proj/tests/test_core.cpp (frobenius_delta,
rescale_dictionary, SolverConfig) and /root/reference/proj/tests/test_kernels.cpp
(is_divergence, solve_h, sample_stats, batch_stats, update_w, majorisation)
against oracle/isnmf_oracle.hpp.  The matrix file round-trip / load-error cases
(test_core.cpp:103-160) belong to io.hpp persistence, out of scope.
The naive helpers below restate tests/oracles.hpp:19-91.
"""
import math

import numpy as np
import pytest

import oracle as O
from oracle import OracleError, random_positive


def rpv(n, seed, lo=0.05, hi=2.0):  # test_kernels.cpp:22-24
    return random_positive(n, 1, seed, lo, hi)[:, 0].copy()


# ---- oracles.hpp:19-91 ----------------------------------------------------------
def is_divergence_naive(y, x, eps):
    r = (eps + np.asarray(y)) / (eps + np.asarray(x))
    return float(np.sum(r - np.log(r) - 1.0))


def objective_naive(v, w, h, eps):
    return sum(is_divergence_naive(v[:, n], w @ h[:, n], eps) for n in range(v.shape[1])) / v.shape[1]


def grid_search_divergence(v, w, eps, lo=1e-3, hi=1e3, points=25, refinements=8):
    k = w.shape[1]
    lo_k = np.full(k, math.log(lo))
    hi_k = np.full(k, math.log(hi))
    best, best_log = math.inf, np.zeros(k)
    for _ in range(refinements):
        t = np.arange(points) / (points - 1)
        axes = [np.exp(lo_k[d] + t * (hi_k[d] - lo_k[d])) for d in range(k)]
        for h in np.array(np.meshgrid(*axes, indexing="ij")).reshape(k, -1).T:
            d_val = is_divergence_naive(v, w @ h, eps)
            if d_val < best:
                best, best_log = d_val, np.log(h)
        span = (hi_k - lo_k) / (points - 1) * 2.0
        lo_k, hi_k = best_log - span, best_log + span
    return best


def aux_partial_fd(a, b, w, rel_step=1e-6):
    d = rel_step * w
    phi = lambda x: a / x + b * x  # noqa: E731
    return (phi(w + d) - phi(w - d)) / (2.0 * d)


# ---- test_core.cpp ----------------------------------------------------------------
def test_frobenius_delta_basics():  # test_core.cpp:32-45
    a = random_positive(4, 3, 1)
    assert O.frobenius_delta(a, a) == 0.0
    b = a.copy()
    b[2, 1] += 3.0
    assert abs(O.frobenius_delta(b, a) - 3.0) < 1e-15
    assert abs(O.frobenius_delta(np.ones((2, 2)), np.zeros((2, 2))) - 2.0) < 1e-15
    with pytest.raises(OracleError) as e:
        O.frobenius_delta(a, np.zeros((3, 3)))
    assert e.value.kind == "ShapeMismatch"


class TestRescaleDictionary:  # test_core.cpp:47-101
    def test_normalized_column_untouched(self):
        w, a, b, _ = O.rescale_dictionary(np.full((4, 1), 0.25), np.full((4, 1), 2.0), np.full((4, 1), 3.0))
        np.testing.assert_allclose(w, 0.25, rtol=1e-12)
        np.testing.assert_allclose(a, 2.0, rtol=1e-12)
        np.testing.assert_allclose(b, 3.0, rtol=1e-12)

    def test_column_2_2_scales_by_4(self):
        w, a, b, _ = O.rescale_dictionary(np.full((2, 1), 2.0), np.full((2, 1), 1.0), np.full((2, 1), 1.0))
        np.testing.assert_allclose(w, 0.5, rtol=1e-12)
        np.testing.assert_allclose(a, 0.25, rtol=1e-12)
        np.testing.assert_allclose(b, 4.0, rtol=1e-12)

    def test_warm_activations_keep_product(self):
        w = random_positive(6, 3, 2)
        h = random_positive(3, 5, 3)
        product = w @ h
        w2, _, _, h2 = O.rescale_dictionary(w, random_positive(6, 3, 4), random_positive(6, 3, 5), h)
        assert np.linalg.norm(w2 @ h2 - product) < 1e-12
        np.testing.assert_allclose(w2.sum(axis=0), 1.0, atol=1e-12)

    def test_idempotent(self):
        d = O.rescale_dictionary(random_positive(5, 2, 6), random_positive(5, 2, 7), random_positive(5, 2, 8))
        again = O.rescale_dictionary(d[0], d[1], d[2])
        for x, y in zip(again[:3], d[:3]):
            assert np.max(np.abs(x - y)) < 1e-12

    def test_preserves_sqrt_a_over_b(self):
        a = random_positive(4, 2, 9)
        b = random_positive(4, 2, 10)
        w2, a2, b2, _ = O.rescale_dictionary(np.sqrt(a / b), a, b)
        assert np.max(np.abs(w2 - np.sqrt(a2 / b2))) < 1e-12

    def test_dead_atom_raises_zero_column(self):
        with pytest.raises(OracleError) as e:
            O.rescale_dictionary(np.zeros((3, 1)), np.zeros((3, 1)), np.zeros((3, 1)))
        assert e.value.kind == "ZeroColumn"


def test_solver_config_validation():  # test_core.cpp:162-181
    O.config_check()
    for kw in (dict(k=0), dict(epsilon=0.0), dict(r=1.5)):
        with pytest.raises(OracleError) as e:
            O.config_check(**kw)
        assert e.value.kind == "NegativeInput"
    assert O.config_check()[0] == 1  # warm default
    assert O.config_check(restart="fresh")[0] == 100
    assert O.config_check(restart="fresh", inner_iters=7)[0] == 7
    eta = O.config_check(F=25, K=4)[1]
    assert abs(eta - 1e-6 * 10.0) <= 1e-12 * 1e-5


# ---- test_kernels.cpp ----------------------------------------------------------------
class TestIsDivergence:  # test_kernels.cpp:28-77
    eps = 1e-12

    def test_zero_iff_equal(self):
        y = rpv(16, 1)
        assert O.is_divergence(y, y, self.eps) == 0.0
        x = y.copy()
        x[3] *= 1.5
        assert O.is_divergence(y, x, self.eps) > 0.0

    def test_frozen_value(self):
        expect = 2.0 * (0.5 + math.log(2.0) - 1.0)  # 0.38629436...
        got = O.is_divergence(np.ones(2), np.full(2, 2.0), 1e-15)
        assert abs(got - expect) <= 1e-9 * expect

    def test_scale_invariance(self):
        lambdas = 0.01 + 100.0 * O.uniform01(7, 50)  # make_engine(7) stream
        for trial in range(50):
            y, x = rpv(8, 100 + trial), rpv(8, 200 + trial)
            d0 = O.is_divergence(y, x, 1e-9)
            d1 = O.is_divergence(lambdas[trial] * y, lambdas[trial] * x, lambdas[trial] * 1e-9)
            assert abs(d1 - d0) <= 1e-10 * abs(d0)

    def test_nonnegative_matches_naive(self):
        for trial in range(100):
            y, x = rpv(12, 300 + trial), rpv(12, 400 + trial)
            d = O.is_divergence(y, x, self.eps)
            assert d >= 0.0
            n = is_divergence_naive(y, x, self.eps)
            assert abs(d - n) <= 1e-10 * abs(n)

    def test_errors(self):
        with pytest.raises(OracleError) as e:
            O.is_divergence(np.ones(3), np.ones(4), self.eps)
        assert e.value.kind == "ShapeMismatch"
        neg = np.ones(3)
        neg[0] = -0.5
        with pytest.raises(OracleError) as e:
            O.is_divergence(neg, neg, self.eps)
        assert e.value.kind == "NegativeInput"
        with pytest.raises(OracleError) as e:
            O.is_divergence(np.ones(3), np.ones(3), 0.0)
        assert e.value.kind == "NegativeInput"


class TestSolveH:  # test_kernels.cpp:79-131
    eps = 1e-12

    def test_exact_reconstruction_fixed_point(self):
        w = random_positive(6, 2, 11)
        h_star = rpv(2, 12)
        h = O.solve_h(w @ h_star, w, h_star, 25, 1e-14)
        assert np.max(np.abs(h - h_star)) < 1e-9

    def test_1d_optimum(self):
        h = O.solve_h(np.array([4.0]), np.array([[2.0]]), np.array([0.3]), 100, self.eps)
        assert abs(h[0] - 2.0) <= 1e-6

    def test_monotone_descent(self):
        w = random_positive(9, 3, 13)
        v = rpv(9, 14)
        h = rpv(3, 15)
        prev = O.is_divergence(v, w @ h, self.eps)
        for _ in range(60):
            h = O.solve_h(v, w, h, 1, self.eps)
            cur = O.is_divergence(v, w @ h, self.eps)
            assert cur <= prev + 1e-10
            prev = cur

    # test_kernels.cpp:112-123 asserts the 100-iteration MM iterate is within
    # 1e-4 of the grid oracle.  With the reference's own update (restated here and
    # cross-checked against a direct numpy MM) that holds for trials 2 and 3 only:
    # trials 0, 1, 4 have an optimum on (or near) the h_k = 0 boundary where MM
    # converges sublinearly (gap 4.7e-3 / 8.4e-4 / 2.5e-3 after 100 iterations).
    # The reference test file is unbuildable here (no Eigen/Catch2), so this
    # golden case was never run upstream; we pin the case as written (strict
    # xfail for the three boundary trials) and the intended property with 1000
    # iterations, where every trial meets the bound.
    @pytest.mark.parametrize("trial", range(5))
    def test_matches_grid_oracle_as_written(self, trial):
        w = random_positive(5, 2, 500 + trial, 0.1, 1.0)
        v = rpv(5, 600 + trial, 0.2, 2.0)
        h = O.solve_h(v, w, np.full(2, 0.5), 100, self.eps)
        got = O.is_divergence(v, w @ h, self.eps)
        assert got >= -1e-12
        ok = got <= grid_search_divergence(v, w, self.eps) + 1e-4
        if trial in (0, 1, 4):
            assert not ok, "boundary trial now converges in 100 iterations: update the pin"
        else:
            assert ok

    def test_matches_grid_oracle_converged(self):
        for trial in range(5):
            w = random_positive(5, 2, 500 + trial, 0.1, 1.0)
            v = rpv(5, 600 + trial, 0.2, 2.0)
            h = O.solve_h(v, w, np.full(2, 0.5), 1000, self.eps)
            got = O.is_divergence(v, w @ h, self.eps)
            assert -1e-12 <= got <= grid_search_divergence(v, w, self.eps) + 1e-4

    def test_rejects_non_positive_init(self):
        with pytest.raises(OracleError) as e:
            O.solve_h(rpv(3, 17), random_positive(3, 2, 16), np.zeros(2), 5, self.eps)
        assert e.value.kind == "NonPositiveInit"


class TestSampleStats:  # test_kernels.cpp:133-165
    def test_1x1_without_floor(self):
        a, b = O.sample_stats(np.array([8.0]), np.array([[2.0]]), np.array([1.0]), 1e-300)
        assert abs(a[0, 0] - 8.0) <= 1e-12 * 8.0
        assert abs(b[0, 0] - 0.5) <= 1e-12 * 0.5
        assert abs(math.sqrt(a[0, 0] / b[0, 0]) - 4.0) <= 1e-12 * 4.0

    def test_1x1_epsilon_one(self):
        a, b = O.sample_stats(np.array([0.0]), np.array([[1.0]]), np.array([1.0]), 1.0)
        assert abs(a[0, 0] - 0.25) <= 1e-12 * 0.25
        assert abs(b[0, 0] - 0.5) <= 1e-12 * 0.5

    def test_fixed_point_identity(self):
        w = random_positive(7, 3, 21)
        h = rpv(3, 22)
        a, b = O.sample_stats(w @ h, w, h, 1e-300)
        assert np.max(np.abs(np.sqrt(a / b) - w)) < 1e-10


class TestBatchStats:  # test_kernels.cpp:167-198
    eps = 1e-12
    v = random_positive(6, 9, 31)
    w = random_positive(6, 3, 32)
    h = random_positive(3, 9, 33)

    def test_single_column_equals_sample_stats(self):
        one = O.batch_stats(self.v[:, :1], self.w, self.h[:, :1], self.eps)
        ref = O.sample_stats(self.v[:, 0], self.w, self.h[:, 0], self.eps)
        assert np.max(np.abs(one[0] - ref[0])) < 1e-14
        assert np.max(np.abs(one[1] - ref[1])) < 1e-14

    def test_equals_sum_over_columns(self):
        fa, fb = O.batch_stats(self.v, self.w, self.h, self.eps)
        sa = sum(O.sample_stats(self.v[:, n], self.w, self.h[:, n], self.eps)[0] for n in range(9))
        sb = sum(O.sample_stats(self.v[:, n], self.w, self.h[:, n], self.eps)[1] for n in range(9))
        assert np.max(np.abs(fa - sa) / sa) < 1e-10
        assert np.max(np.abs(fb - sb) / sb) < 1e-10

    def test_recovers_w_on_exact_factorisation(self):
        a, b = O.batch_stats(self.w @ self.h, self.w, self.h, 1e-300)
        assert np.max(np.abs(np.sqrt(a / b) - self.w)) < 1e-10


class TestUpdateW:  # test_kernels.cpp:200-259
    def test_frozen_values(self):
        a = np.full((3, 2), 0.7)
        assert np.max(np.abs(O.update_w(a, a, np.full((3, 2), 0.123)) - 1.0)) < 1e-15
        assert abs(O.update_w(np.array([[4.0]]), np.array([[1.0]]), np.ones((1, 1)))[0, 0] - 2.0) <= 2e-15

    def test_dead_entries_keep_previous(self):
        a, b = np.zeros((2, 1)), np.zeros((2, 1))
        a[0, 0], b[0, 0] = 1.0, 4.0
        w = O.update_w(a, b, np.array([[0.3], [0.7]]))
        assert abs(w[0, 0] - 0.5) <= 0.5e-15
        assert w[1, 0] == 0.7

    def test_inconsistent(self):
        with pytest.raises(OracleError) as e:
            O.update_w(np.ones((1, 1)), np.zeros((1, 1)), np.ones((1, 1)))
        assert e.value.kind == "InconsistentStats"

    def test_perturbation_increases_aux(self):
        rng = np.random.default_rng(55)
        for trial in range(20):
            a, b = random_positive(4, 3, 700 + trial), random_positive(4, 3, 800 + trial)
            w = O.update_w(a, b, np.ones((4, 3)))
            base = O.aux_value(a, b, w)
            for _ in range(10):
                i, j = rng.integers(4), rng.integers(3)
                wp = w.copy()
                wp[i, j] *= 1.01 if rng.random() < 0.5 else 0.99
                assert O.aux_value(a, b, wp) > base

    def test_fd_gradient_vanishes(self):
        for trial in range(20):
            a, b = random_positive(5, 2, 900 + trial), random_positive(5, 2, 950 + trial)
            w = O.update_w(a, b, np.ones((5, 2)))
            worst = max(abs(aux_partial_fd(a[i, j], b[i, j], w[i, j])) for i in range(5) for j in range(2))
            assert worst < 1e-6


class TestMajorisation:  # test_kernels.cpp:261-303
    def test_frozen_1x1(self):
        one = np.ones((1, 1))
        assert abs(O.aux_value(one, one, one) - 2.0) <= 2e-15

    def test_objective_vanishes_on_exact(self):
        w, h = random_positive(5, 2, 61), random_positive(2, 7, 62)
        o = O.objective(w @ h, w, h, 1e-300)
        assert o < 1e-12
        assert abs(o + 1.0 - 1.0) <= 1e-9

    def test_objective_matches_naive(self):
        v, w, h = random_positive(6, 5, 63), random_positive(6, 2, 64), random_positive(2, 5, 65)
        n = objective_naive(v, w, h, 1e-12)
        assert abs(O.objective(v, w, h, 1e-12) - n) <= 1e-10 * n

    def test_bound_with_equality_at_anchor(self):
        eps = 1e-12
        for trial in range(10):
            f, k, n = 8, 3, 6
            v = random_positive(f, n, 1000 + trial)
            wu = random_positive(f, k, 1100 + trial)
            h = random_positive(k, n, 1200 + trial)
            a, b = O.batch_stats(v, wu, h, eps)
            c = O.aux_constant(v, wu, h, eps)
            n_obj = n * O.objective(v, wu, h, eps)
            assert abs(O.aux_value(a, b, wu) + c - n_obj) <= 1e-8 * abs(n_obj)
            for probe in range(30):
                wp = random_positive(f, k, 2000 + 100 * trial + probe, 0.02, 3.0)
                lhs = O.aux_value(a, b, wp) + c
                rhs = n * O.objective(v, wp, h, eps)
                assert lhs >= rhs - 1e-9 * abs(rhs)
