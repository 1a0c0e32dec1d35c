"""GPU parity of the batch O(FKN) path (batch.hpp:84-143) against the oracle:
per-epoch objective and final W within 1e-4 relative (BASELINE config 2 shape,
reduced N so the fp64 oracle finishes in seconds), monotone descent, the
batch == online equivalence on the device, and error mapping."""
import numpy as np
import pytest

import oracle as O
import paper_1106_4198_b200 as E
from tools.synth import spectrogram_np, w_init

pytestmark = pytest.mark.gpu
RTOL = 1e-4


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


@pytest.mark.parametrize("F,K,N,epochs", [(513, 50, 2000, 5), (257, 10, 3000, 12), (40, 3, 77, 20),
                                          (129, 96, 1500, 4)])  # K = 96: tensor-pipe kernel
def test_batch_matches_oracle(F, K, N, epochs):
    v = spectrogram_np(F, K, N, seed=21)
    rng = np.random.default_rng(22)
    w0 = rng.uniform(0.1, 1.0, size=(F, K))
    h0 = rng.uniform(0.1, 1.0, size=(K, N))
    got = E.batch_train(v, w0, h0, epochs)
    ref = O.batch_train(v.astype(np.float64), w0, h0, epochs)
    assert got["epochs"] == ref["epochs"] == epochs
    assert rel(got["initial_obj"], ref["initial_obj"]) < RTOL
    assert rel(got["obj"], ref["obj"]) < RTOL
    assert rel(got["w"], ref["w"]) < 1e-3  # W after several epochs accumulates fp32 drift
    assert np.all(np.diff(np.concatenate([[got["initial_obj"]], got["obj"]])) <= 1e-6 * got["initial_obj"])


def test_batch_multi_tile_ctas_match_oracle_and_reproduce():
    """N large enough that every CTA of the persistent K1M launch owns several frame tiles
    (148 CTAs x 32 frames per tile): the CTA's statistics plane is written by a bulk store for
    its first tile and accumulated by cp.reduce.async.bulk adds for the others, in tile order —
    per-epoch objectives and W against the oracle, and two runs bitwise identical."""
    F, K, N, epochs = 100, 20, 3 * 148 * 32 + 1234, 3  # 3-4 tiles per CTA, ragged last tile
    v = spectrogram_np(F, K, N, seed=31)
    rng = np.random.default_rng(32)
    w0 = rng.uniform(0.1, 1.0, size=(F, K))
    h0 = rng.uniform(0.1, 1.0, size=(K, N))
    got = E.batch_train(v, w0, h0, epochs)
    ref = O.batch_train(v.astype(np.float64), w0, h0, epochs)
    assert rel(got["initial_obj"], ref["initial_obj"]) < RTOL
    assert rel(got["obj"], ref["obj"]) < RTOL
    assert rel(got["w"], ref["w"]) < 1e-3
    again = E.batch_train(v, w0, h0, epochs)
    assert np.array_equal(got["w"], again["w"]) and np.array_equal(got["obj"], again["obj"])
    assert np.array_equal(got["h"], again["h"])


def test_batch_eta_stop_and_final_objective():
    F, K, N = 64, 4, 500
    v = spectrogram_np(F, K, N, seed=5)
    w0 = w_init(F, K, 6) * 3.0
    h0 = np.full((K, N), 0.5)
    got = E.batch_train(v, w0, h0, 200, eta=1e-4)
    ref = O.batch_train(v.astype(np.float64), w0, h0, 200, eta=1e-4)
    assert abs(got["epochs"] - ref["epochs"]) <= 1
    n = min(got["epochs"], ref["epochs"])
    assert rel(got["obj"][:n], ref["obj"][:n]) < RTOL


def test_batch_equals_online_on_device():  # SPEC.md:413 criterion 5, through the engine
    F, K, N, E_ = 20, 4, 50, 6
    v = spectrogram_np(F, K, N, seed=11)
    w0 = w_init(F, K, 12)
    h0 = O.default_h0(v.astype(np.float64), w0)
    batch = E.batch_train(v, w0, h0, E_)
    eng = E.Online(F, K, N, 1, restart="warm", n_store=N)
    eng.set_dictionary(w0, np.zeros((F, K)), np.zeros((F, K)))
    eng.set_counters(0, 0, 0.0)
    eng.set_warm_h(h0)
    for _ in range(E_):
        eng.run(v, index=np.arange(N))
    assert rel(eng.state()["w"], batch["w"]) < RTOL


def test_batch_errors():
    v = np.ones((5, 4), np.float32)
    with pytest.raises(E.EngineError) as e:
        E.batch_train(v, np.zeros((5, 2)), np.ones((2, 4)), 3)
    assert e.value.kind == "NonPositiveInit"
    h0 = np.ones((2, 4))
    h0[1, 2] = 0.0  # checked on the device while H0 is converted
    with pytest.raises(E.EngineError) as e:
        E.batch_train(v, np.ones((5, 2)), h0, 3)
    assert e.value.kind == "NonPositiveInit"
    h0[1, 2] = np.nan
    with pytest.raises(E.EngineError) as e:
        E.batch_train(v, np.ones((5, 2)), h0, 3)
    assert e.value.kind == "NonPositiveInit"
    out = E.batch_train(v, np.ones((5, 2)), np.ones((2, 4)), 3)  # the context is usable afterwards
    assert out["epochs"] == 3
