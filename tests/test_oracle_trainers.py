"""Holds the oracle's online / batch trainers to the SPEC.md examples and
acceptance properties (the reference ships no trainer tests: proj/tests/
CMakeLists.txt:7-10 lists test_online.cpp / test_batch.cpp, absent — so beyond
these properties the trainer restatement is "parity unpinned").
"""
import numpy as np
import pytest

import oracle as O
from oracle import random_positive


def normalized(w):
    return w / w.sum(axis=0, keepdims=True)


def test_batch_monotone_descent():  # SPEC.md:409 criterion 2 (50x200, K=5, 100 epochs)
    v = random_positive(50, 200, 1, 0.01, 1.0)
    w0 = random_positive(50, 5, 2, 0.1, 1.0)
    h0 = random_positive(5, 200, 3, 0.1, 1.0)
    out = O.batch_train(v, w0, h0, 100)
    obj = np.concatenate([[out["initial_obj"]], out["obj"]])
    assert out["epochs"] == 100
    assert np.all(np.diff(obj) <= 1e-9 * obj[:-1])
    np.testing.assert_allclose(out["w"].sum(axis=0), 1.0, atol=1e-12)


def test_batch_exact_fixed_point():  # V = W*H* exact, start at the optimum
    w = normalized(random_positive(8, 3, 4))
    h = random_positive(3, 20, 5)
    out = O.batch_train(w @ h, w, h, 5, eps=1e-300, eta=1e-10)
    assert out["epochs"] == 1
    assert out["last_delta"] < 1e-10


@pytest.mark.parametrize("permute", [False, True])
def test_online_equals_batch(permute):  # SPEC.md:413 criterion 5 (F=20, K=4, N=50, 10 epochs)
    F, K, N, E = 20, 4, 50, 10
    v = random_positive(F, N, 11, 0.01, 1.0)
    w0 = normalized(random_positive(F, K, 12, 0.1, 1.0))
    h0 = O.default_h0(v, w0)
    batch = O.batch_train(v, w0, h0, E)
    on = O.Online(w0, beta=N, r=0.0, inner_iters=1, restart="warm", init_stats_weight=0.0,
                  dataset_size=N, dataset=v)
    assert on.state()["rho"] == 0.0
    for epoch in range(E):
        order = O.cycle_permutation(7, epoch, N) if permute else np.arange(N, dtype=np.uint64)
        on.run(v[:, order.astype(np.int64)], index=order)
        w_on = on.state()["w"]
        # batch trainer's W after `epoch+1` epochs
        w_b = O.batch_train(v, w0, h0, epoch + 1)["w"]
        assert np.max(np.abs(w_on - w_b) / np.abs(w_b)) < 1e-8
    np.testing.assert_allclose(on.state()["w"], batch["w"], rtol=1e-8)


def test_beta_gating_and_commit():
    w0 = normalized(random_positive(6, 2, 21))
    v = random_positive(6, 2, 22)
    on = O.Online(w0, beta=2, r=1.0, inner_iters=5, restart="fresh", dataset_size=2)
    on.step(v[:, 0], 0)
    s = on.state()
    assert s["commits"] == 0 and np.array_equal(s["w"], w0) and s["pending_count"] == 1
    on.step(v[:, 1], 1)
    s = on.state()
    assert s["commits"] == 1 and not np.array_equal(s["w"], w0)
    assert np.all(s["pending_a"] == 0) and s["pending_count"] == 0


def test_single_step_w_becomes_4_before_rescale():  # SPEC.md:254 (pre-rescale reading)
    # F=K=1, W=2, h forced to 1 (warm store), v=8, beta=1, rho=1, A0=B0=0.
    on = O.Online(np.ones((1, 1)), beta=1, r=1.0, inner_iters=1, restart="warm", init_stats_weight=0.0,
                  dataset_size=1, dataset=np.array([[8.0]]), epsilon=1e-300)
    on.set(w=np.array([[2.0]]), warm_h=np.ones((1, 1)), t=0, commits=0)
    # one MM iteration moves h; pin the SPEC example through the stats instead:
    a, b = O.sample_stats(np.array([8.0]), np.array([[2.0]]), np.array([1.0]), 1e-300)
    assert abs(np.sqrt(a[0, 0] / b[0, 0]) - 4.0) < 1e-12
    on.run(np.array([[8.0]]), index=np.array([0], dtype=np.uint64))
    assert abs(on.state()["w"][0, 0] - 1.0) < 1e-15  # l1 rescale at F=1 forces W=1 (model.hpp:79-81)


def test_rho_one_accumulates_monotonically():
    F, K, N = 10, 3, 40
    v = random_positive(F, N, 31, 0.01, 1.0)
    w0 = normalized(random_positive(F, K, 32, 0.1, 1.0))
    on = O.Online(w0, beta=10, r=1.0, inner_iters=3, restart="fresh", seed=5, dataset_size=N)
    prev_b = on.state()["b"].copy()
    for c in range(4):
        on.run(v[:, 10 * c:10 * c + 10], index_base=10 * c)
        s = on.state()
        # B is compensated by the rescale (B *= s): compare the unscaled sums via A/B invariance
        assert s["commits"] == c + 1
        assert np.all(np.isfinite(s["w"]))
        prev_b = s["b"]
    assert prev_b.shape == (F, K)


def test_rho_from_r():  # r=0.49, beta=N/2 -> rho=0.7
    on = O.Online(normalized(np.ones((3, 1))), beta=5, r=0.49, restart="fresh", dataset_size=10)
    assert abs(on.state()["rho"] - 0.7) < 1e-15
    on2 = O.Online(normalized(np.ones((3, 1))), beta=5, r=0.49, restart="fresh")
    assert on2.state()["rho"] == 1.0  # unsized stream (online.hpp:274-277)


def test_budget_zero_returns_w0():
    w0 = normalized(random_positive(5, 2, 41))
    on = O.Online(w0, beta=2, restart="fresh", budget=0, dataset_size=4)
    tt, _ = on.run(random_positive(5, 4, 42))
    assert len(tt) == 0 and np.array_equal(on.state()["w"], w0)


def test_leftover_frames_accumulate_but_do_not_commit():  # online.hpp:386-388
    w0 = normalized(random_positive(5, 2, 51))
    on = O.Online(w0, beta=4, r=1.0, inner_iters=2, restart="fresh", dataset_size=10)
    tt, to = on.run(random_positive(5, 10, 52))
    s = on.state()
    assert s["commits"] == 2 and s["t"] == 10 and s["pending_count"] == 2
    assert list(tt) == [4, 8] and np.all(s["pending_a"] > 0)


def test_init_errors():  # online.hpp:258-265, 279-280
    with pytest.raises(O.OracleError) as e:
        O.Online(np.ones((3, 2)), beta=2, restart="fresh")
    assert e.value.kind == "NonPositiveInit"
    with pytest.raises(O.OracleError) as e:
        O.Online(normalized(np.ones((3, 2))), beta=2, restart="warm")
    assert e.value.kind == "EmptyDataset"


def test_cycle_permutation_is_a_permutation():  # online.hpp:79-87
    p = O.cycle_permutation(3, 0, 100)
    assert sorted(p.tolist()) == list(range(100))
    assert not np.array_equal(p, O.cycle_permutation(3, 1, 100))
    assert np.array_equal(p, O.cycle_permutation(3, 0, 100))


def test_heldout_init_stream_and_objective():  # harness.hpp:17-37
    rng = np.random.default_rng(5)
    w = rng.uniform(0.1, 1.0, (33, 4))
    w /= w.sum(axis=0)
    t = rng.uniform(0.01, 2.0, (33, 20))
    h0 = O.heldout_h0(w, t, 1e-12, 0x45)
    u = O.uniform01(O.mix_seed(0x45, 0xE7A1), 4 * 20)  # one stream, column-major fill
    scale = max(t.mean(), 1e-12) / (4 * w.mean())
    assert np.allclose(h0, scale * (1.0 - u).reshape(20, 4).T, rtol=1e-13, atol=0)
    d0 = O.evaluate_heldout(w, t, 1e-12, 0, 0x45)
    assert abs(d0 - O.objective(t, w, h0, 1e-12)) <= 1e-12 * d0
    d = [O.evaluate_heldout(w, t, 1e-12, it, 0x45) for it in (1, 10, 100)]
    assert d0 > d[0] > d[1] > d[2] > 0.0
    with pytest.raises(O.OracleError):
        O.evaluate_heldout(w, t[:5], 1e-12)
