"""K1C — the 2-SM tcgen05 solve for K <= 56 (csrc/kernels_tc.cuh) — against the oracle
and against K1M (the mma.sync kernel it replaces at config 3).

The shapes the engine routes to K1C (F in (384, 520], 17 <= K <= 56, >= 40 frames per
pair of SMs) are covered by the generic online suites too (test_gpu_online,
test_gpu_trajectory, test_gpu_longrun, test_gpu_fullsize, test_gpu_ref_trainers); here:
the routing itself, state injection at F = 512 (no tail row) and F = 520 (8 tail rows),
K not a multiple of 8, partial pairs (nframes not a multiple of the pair size), forced
small mini-batches, fresh restarts, and K1C vs K1M on the same state (1e-4, the
north-star tolerance).
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


def injected(F, K, beta, iters, restart, pair, seed=3, nmb=1, rho=0.95967):
    rng = np.random.default_rng(seed)
    N = beta * nmb
    v = spectrogram_np(F, K, N, seed=seed + 1)
    w = w_init(F, K, seed=seed + 2)
    a = rng.uniform(0.5, 2.0, size=(F, K)) * w * w
    b = rng.uniform(0.5, 2.0, size=(F, K))
    eng = E.Online(F, K, beta, iters, restart=restart, seed=seed, n_store=N if restart == "warm" else 0, pair=pair)
    eng.set_dictionary(w, a, b)
    eng.set_counters(0, 0, rho)
    orc = O.Online(w, beta=beta, r=1.0, inner_iters=iters, restart=restart, seed=seed, dataset_size=N,
                   dataset=v.astype(np.float64) if restart == "warm" else None)
    orc.set(a=a, b=b, rho=rho, t=0, commits=0)
    if restart == "warm":
        h0 = rng.gamma(2.0, 0.5, size=(K, N)) + 1e-2
        eng.set_warm_h(h0)
        orc.set(warm_h=h0, rho=rho, t=0, commits=0)
    return eng, orc, v


def check(eng, orc, v, restart):
    orc.run(v.astype(np.float64))
    eng.run(v)
    so = orc.state(warm_h=restart == "warm")
    se = eng.state(warm_h=restart == "warm")
    for k in ("w", "a", "b"):
        assert rel(se[k], so[k]) < RTOL, (k, rel(se[k], so[k]))
    assert se["commits"] == so["commits"]
    assert rel(se["last_minibatch_obj"], so["last_minibatch_obj"]) < RTOL
    if restart == "warm":
        assert rel(se["warm_h"], so["warm_h"]) < RTOL
    return se


def test_config3_routes_to_k1c():
    assert E.Online(513, 50, 4096, 10, n_store=4096).solver() == "K1C"
    assert E.Online(513, 50, 4096, 10, n_store=4096, pair=False).solver() == "K1M"
    assert E.Online(257, 10, 100, 5, n_store=100).solver() != "K1C"  # F too small for a pair


@pytest.mark.parametrize("restart", ["warm", "fresh"])
@pytest.mark.parametrize("F,K,beta,iters", [
    (513, 50, 4096, 10),   # config 3: 74 pairs of 56 frames, one tail row
    (512, 50, 4096, 10),   # no tail row
    (520, 43, 3000, 7),    # 8 tail rows, K not a multiple of 8, partial last pair
    (450, 24, 3100, 4),    # rows of CTA 1 partly past F
])
def test_k1c_state_injection(F, K, beta, iters, restart):
    eng, orc, v = injected(F, K, beta, iters, restart, pair=None)
    assert eng.solver() == "K1C"
    check(eng, orc, v, restart)


@pytest.mark.parametrize("beta", [100, 700])
def test_k1c_forced_small_minibatches(beta):
    # pairs of 8 / 16 frames, two mini-batches (a commit between them)
    eng, orc, v = injected(513, 50, beta, 10, "warm", pair=True, nmb=2)
    assert eng.solver() == "K1C"
    check(eng, orc, v, "warm")


def test_k1c_matches_k1m():
    F, K, beta, iters = 513, 50, 4096, 10
    res = {}
    for pair in (True, False):
        eng, orc, v = injected(F, K, beta, iters, "warm", pair=pair, nmb=2)
        eng.run(v)
        res[pair] = eng.state(warm_h=True)
    for k in ("w", "a", "b", "warm_h"):
        assert rel(res[True][k], res[False][k]) < RTOL, k
    assert rel(res[True]["last_minibatch_obj"], res[False]["last_minibatch_obj"]) < RTOL


def test_k1c_bitwise_reproducible():
    out = []
    for _ in range(2):
        eng, orc, v = injected(513, 50, 4096, 10, "warm", pair=None, nmb=2)
        eng.run(v)
        out.append(eng.state(warm_h=True))
    for k in ("w", "a", "b", "warm_h"):
        assert np.array_equal(out[0][k], out[1][k]), k
