"""K1M numerics under wide dynamic ranges (3xTF32 splits of every operand, the fp32
q = (v+eps)/Lam^2): one mini-batch from an injected state at the config-3 shape
against the fp64 oracle, at the north-star 1e-4 relative tolerance.

* V: silent frames at the 1e-9 floor next to frames scaled by 1e6;
* W: entries spread over six decades (column-normalised);
* warm H: entries spread over nine decades.
"""
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


def one_minibatch(v, w, a, b, h0, iters=10, rho=0.95967):
    F, K = w.shape
    beta = v.shape[1]
    eng = E.Online(F, K, beta, iters, restart="warm", n_store=beta)
    eng.set_dictionary(w, a, b)
    eng.set_counters(0, 0, rho)
    eng.set_warm_h(h0)
    orc = O.Online(w, beta=beta, r=1.0, inner_iters=iters, restart="warm", dataset_size=beta,
                   dataset=v.astype(np.float64))
    orc.set(w=w, a=a, b=b, rho=rho, t=0, commits=0, warm_h=h0)
    orc.run(v.astype(np.float64))
    eng.run(v)
    se, so = eng.state(warm_h=True), orc.state(warm_h=True)
    errs = {k: rel(se[k], so[k]) for k in ("w", "a", "b", "warm_h")}
    errs["obj"] = rel(se["last_minibatch_obj"], so["last_minibatch_obj"])
    eng.close()
    return errs


F, K, BETA = 513, 50, 4096


def base_state(seed):
    rng = np.random.default_rng(seed)
    w = w_init(F, K, seed)
    a = rng.uniform(0.5, 2.0, size=(F, K)) * w * w
    b = rng.uniform(0.5, 2.0, size=(F, K))
    h0 = rng.gamma(2.0, 0.5, size=(K, BETA)) + 1e-2
    return rng, w, a, b, h0


def test_silent_and_loud_frames():
    rng, w, a, b, h0 = base_state(31)
    v = spectrogram_np(F, K, BETA, seed=32)
    v[:, ::5] = 1e-9                        # silent frames
    v[:, 1::7] *= np.float32(1e6)           # loud frames
    errs = one_minibatch(v, w, a, b, h0)
    assert max(errs.values()) < RTOL, errs


def test_dictionary_over_six_decades():
    rng, _, _, _, h0 = base_state(41)
    w = 10.0 ** rng.uniform(-6.0, 0.0, size=(F, K))
    w /= w.sum(axis=0, keepdims=True)
    a = rng.uniform(0.5, 2.0, size=(F, K)) * w * w
    b = rng.uniform(0.5, 2.0, size=(F, K))
    v = spectrogram_np(F, K, BETA, seed=42)
    errs = one_minibatch(v, np.asfortranarray(w), a, b, h0)
    assert max(errs.values()) < RTOL, errs


def test_activations_over_nine_decades():
    rng, w, a, b, _ = base_state(51)
    h0 = 10.0 ** rng.uniform(-6.0, 3.0, size=(K, BETA))
    v = spectrogram_np(F, K, BETA, seed=52)
    errs = one_minibatch(v, w, a, b, h0)
    assert max(errs.values()) < RTOL, errs
