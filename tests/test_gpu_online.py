"""GPU parity of the online hot path (online.hpp:254-419) against the oracle.

(1) State injection: the same state (W, A, B, rho, warm h / fresh seed) is
    loaded into the engine and the oracle, one mini-batch is run, and the H
    block, A, B, W after the commit and the mini-batch objective are compared
    (relative 1e-4, the north_star tolerance).
(2) Free-running: BASELINE config 0 (F=257, K=10, beta=100, I=5, N=1e4, 1 pass)
    and a 20-mini-batch prefix of config 1 end to end: final W, A, B and the
    final objective within 1e-4 relative.
(3) Reproducibility: two runs are bitwise identical (fixed-order reductions).
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


def make_pair(F, K, beta, iters, N, restart="warm", seed=7, rho=1.0, a0=1e-3, v=None, generic=False):
    """Engine + oracle with the BASELINE initial state (A0 = B0 = a0, warm_h = 1)."""
    w0 = w_init(F, K, seed)
    v = spectrogram_np(F, K, N, seed=seed + 1) if v is None else v
    eng = E.Online(F, K, beta, iters, restart=restart, seed=seed, n_store=N if restart == "warm" else 0,
                   generic=generic)
    eng.set_dictionary(w0, np.full((F, K), a0), np.full((F, K), a0))
    eng.set_counters(0, 0, rho)
    orc = O.Online(w0, beta=beta, r=1.0, inner_iters=iters, restart=restart, seed=seed, dataset_size=N,
                   dataset=v.astype(np.float64) if restart == "warm" else None)
    orc.set(a=np.full((F, K), a0), b=np.full((F, K), a0), rho=rho, t=0, commits=0,
            warm_h=np.ones((K, N)) if restart == "warm" else None)
    if restart == "warm":
        eng.fill_warm_h(1.0)
    return eng, orc, v


def compare_state(eng, orc, tol=RTOL, keys=("w", "a", "b")):
    se, so = eng.state(), orc.state()
    for k in keys:
        assert rel(se[k], so[k]) < tol, (k, rel(se[k], so[k]))
    assert se["t"] == so["t"] and se["commits"] == so["commits"]
    return se, so


@pytest.mark.parametrize("restart", ["warm", "fresh"])
@pytest.mark.parametrize("F,K,beta,iters", [(257, 10, 100, 5), (513, 20, 1000, 10), (513, 50, 4096, 10)])
def test_state_injection_one_minibatch(F, K, beta, iters, restart):
    rng = np.random.default_rng(F + K)
    N = beta
    eng, orc, v = make_pair(F, K, beta, iters, N, restart=restart, rho=0.95967)
    # inject a non-trivial state: W ~ normalised U, A, B ~ positive, warm h ~ Gamma
    w = w_init(F, K, seed=99)
    a = rng.uniform(0.5, 2.0, size=(F, K)) * w * w
    b = rng.uniform(0.5, 2.0, size=(F, K))
    eng.set_dictionary(w, a, b)
    orc.set(w=w, a=a, b=b, rho=0.95967, t=0, commits=0)
    if restart == "warm":
        h0 = rng.gamma(2.0, 0.5, size=(K, N)) + 1e-2
        eng.set_warm_h(h0)
        orc.set(warm_h=h0, rho=0.95967, t=0, commits=0)
    orc.run(v.astype(np.float64))
    eng.run(v)
    so = orc.state(warm_h=restart == "warm")
    se = eng.state(warm_h=restart == "warm")
    for k in ("w", "a", "b"):
        assert rel(se[k], so[k]) < RTOL, (k, rel(se[k], so[k]))
    assert se["commits"] == so["commits"] == 1
    assert rel(se["last_minibatch_obj"], so["last_minibatch_obj"]) < RTOL
    if restart == "warm":
        assert rel(se["warm_h"], so["warm_h"]) < RTOL
    assert abs(se["last_delta"] - so["last_delta"]) <= RTOL * so["last_delta"] + 1e-6 * np.linalg.norm(w)


def test_free_running_config0():
    c = dict(F=257, K=10, beta=100, iters=5, N=10_000)
    eng, orc, v = make_pair(c["F"], c["K"], c["beta"], c["iters"], c["N"])
    tt, to = orc.run(v.astype(np.float64))
    eng.run(v)
    compare_state(eng, orc)
    s, o, sec = eng.trace()
    assert list(s) == list(tt) and len(s) == 100
    assert rel(o, to) < RTOL
    assert rel(o[-1], to[-1]) < RTOL  # final objective
    assert np.all(np.diff(sec) >= 0)


def test_free_running_config1_prefix():
    F, K, beta, iters, N = 513, 20, 1000, 10, 20_000
    eng, orc, v = make_pair(F, K, beta, iters, N)
    tt, to = orc.run(v.astype(np.float64))
    eng.run(v)
    compare_state(eng, orc)
    _, o, _ = eng.trace()
    assert rel(o, to) < RTOL


def test_free_running_fresh_and_forgetting():
    F, K, beta, iters, N = 129, 8, 64, 20, 64 * 12 + 17
    eng, orc, v = make_pair(F, K, beta, iters, N, restart="fresh", rho=0.7)
    orc.run(v.astype(np.float64))
    eng.run(v)
    se, so = compare_state(eng, orc, keys=("w", "a", "b", "pending_a", "pending_b"))
    assert se["pending_count"] == so["pending_count"] == 17


def test_reproducible_bitwise():
    F, K, beta, iters, N = 257, 10, 100, 5, 2000
    outs = []
    for _ in range(2):
        eng, _, v = make_pair(F, K, beta, iters, N)
        eng.run(v)
        outs.append(eng.state(warm_h=True))
    for k in ("w", "a", "b", "warm_h"):
        assert np.array_equal(outs[0][k], outs[1][k])


def test_host_and_device_frames_agree():
    import torch
    F, K, beta, iters, N = 257, 10, 100, 5, 3000
    e1, _, v = make_pair(F, K, beta, iters, N)
    e1.run(v)
    e2, _, _ = make_pair(F, K, beta, iters, N, v=v)
    vt = torch.from_numpy(np.ascontiguousarray(v.T)).cuda()
    e2.run(vt)
    e3 = E.Online(F, K, beta, iters, restart="warm", n_store=N, max_chunk=700)  # unaligned chunks
    e3.set_dictionary(w_init(F, K, 7), np.full((F, K), 1e-3), np.full((F, K), 1e-3))
    e3.fill_warm_h(1.0)
    e3.run(torch.from_numpy(np.ascontiguousarray(v.T)).pin_memory())
    s1, s2, s3 = e1.state(), e2.state(), e3.state()
    for k in ("w", "a", "b"):
        assert np.array_equal(s1[k], s2[k]) and np.array_equal(s1[k], s3[k])


def test_budget_eta_and_cycling_indices():
    F, K, beta, iters, N = 65, 4, 16, 3, 64
    v = spectrogram_np(F, K, N, seed=3)
    w0 = w_init(F, K, 5)
    for eta in (0.0, 5e-3):
        eng = E.Online(F, K, beta, iters, restart="warm", n_store=N)
        eng.set_dictionary(w0, w0 * w0, np.ones((F, K)))
        eng.set_counters(0, 0, 1.0)
        eng.fill_warm_h(0.3)
        orc = O.Online(w0, beta=beta, r=1.0, inner_iters=iters, restart="warm", eta=eta, budget=150,
                       dataset_size=N, dataset=v.astype(np.float64))
        orc.set(warm_h=np.full((K, N), 0.3), rho=1.0, t=0, commits=0)
        # three cycles of the reference CyclingSource order (online.hpp:79-87)
        order = np.concatenate([O.cycle_permutation(11, c, N) for c in range(3)]).astype(np.int64)
        orc.run(v[:, order].astype(np.float64), index=order.astype(np.uint64))
        stopped = eng.run(v[:, order], index=order, budget=150, eta=eta)
        se, so = eng.state(warm_h=True), orc.state(warm_h=True)
        assert se["t"] == so["t"] and se["commits"] == so["commits"]
        assert stopped == (eta > 0 and so["t"] < 150)
        for k in ("w", "a", "b", "warm_h", "pending_a"):
            assert rel(se[k], so[k]) < RTOL, (eta, k)


def test_errors_map_to_reference_types():
    F, K = 17, 2
    with pytest.raises(E.EngineError) as e:
        E.Online(F, K, 4, 1, restart="warm", n_store=0)
    assert e.value.kind == "EmptyDataset"
    eng = E.Online(F, K, 4, 1, restart="warm", n_store=3)
    eng.set_dictionary(w_init(F, K, 1), np.ones((F, K)), np.ones((F, K)))
    eng.fill_warm_h(1.0)
    with pytest.raises(E.EngineError) as e:
        eng.run(np.ones((F, 4), np.float32), index=np.arange(4))  # index 3 outside the store
    assert e.value.kind == "ShapeMismatch"
    eng = E.Online(F, K, 4, 1, restart="warm", n_store=4)
    eng.set_dictionary(w_init(F, K, 1), np.ones((F, K)), np.ones((F, K)))
    eng.fill_warm_h(0.0)
    with pytest.raises(E.EngineError) as e:
        eng.run(np.ones((F, 4), np.float32))
    assert e.value.kind == "NonPositiveInit"


@pytest.mark.parametrize("F,K,beta,iters,N,restart", [
    (1025, 256, 256, 8, 512, "warm"),   # config 4 shape (F, K, I), reduced beta / N for the fp64 oracle
    (129, 80, 96, 4, 300, "fresh"),
    (33, 3, 10, 5, 47, "warm"),
])
def test_generic_large_k_kernel(F, K, beta, iters, N, restart):
    """The W-streaming generic kernel (K > 64 or forced) against the oracle."""
    eng, orc, v = make_pair(F, K, beta, iters, N, restart=restart, rho=0.9, generic=True)
    orc.run(v.astype(np.float64))
    eng.run(v)
    keys = ("w", "a", "b", "pending_a", "pending_b") + (("warm_h",) if restart == "warm" else ())
    se, so = eng.state(warm_h=restart == "warm"), orc.state(warm_h=restart == "warm")
    for k in keys:
        assert rel(se[k], so[k]) < RTOL, (k, rel(se[k], so[k]))
    assert se["commits"] == so["commits"] and se["pending_count"] == so["pending_count"]
    assert rel(se["last_minibatch_obj"], so["last_minibatch_obj"]) < RTOL


def test_generic_and_tiled_kernels_agree():
    F, K, beta, iters, N = 257, 10, 100, 5, 1000
    e1, _, v = make_pair(F, K, beta, iters, N)
    e2, _, _ = make_pair(F, K, beta, iters, N, v=v, generic=True)
    e1.run(v)
    e2.run(v)
    s1, s2 = e1.state(), e2.state()
    for k in ("w", "a", "b"):
        assert rel(s1[k], s2[k]) < 1e-5


@pytest.mark.parametrize("F,K,beta,iters,N,restart", [
    (1025, 256, 256, 8, 512, "warm"),   # config-4 dictionary shape, 8 frames per CTA
    (129, 80, 96, 4, 300, "fresh"),     # K <= 128: one m-block per warp
    (129, 256, 8192, 2, 8192, "warm"),  # config-4 frames per CTA (56), ragged last window
    (1025, 200, 2048, 3, 2048, "fresh"),  # K padded to 256
    (129, 200, 9472, 2, 9472, "warm"),    # 64 frames per CTA: the mma.sync kernel (tcgen05 variant holds <= 56)
])
def test_large_k_tensor_kernel(F, K, beta, iters, N, restart):
    """The tensor-pipe kernel (3xTF32 mma.sync, 64 < K <= 256) against the oracle."""
    eng, orc, v = make_pair(F, K, beta, iters, N, restart=restart, rho=0.9)
    orc.run(v.astype(np.float64))
    eng.run(v)
    keys = ("w", "a", "b", "pending_a", "pending_b") + (("warm_h",) if restart == "warm" else ())
    se, so = eng.state(warm_h=restart == "warm"), orc.state(warm_h=restart == "warm")
    for k in keys:
        assert rel(se[k], so[k]) < RTOL, (k, rel(se[k], so[k]))
    assert se["commits"] == so["commits"] and se["pending_count"] == so["pending_count"]
    assert rel(se["last_minibatch_obj"], so["last_minibatch_obj"]) < RTOL


def test_large_k_tensor_and_generic_kernels_agree():
    F, K, beta, iters, N = 257, 128, 512, 4, 1024
    e1, _, v = make_pair(F, K, beta, iters, N)
    e2, _, _ = make_pair(F, K, beta, iters, N, v=v, generic=True)
    e1.run(v)
    e2.run(v)
    s1, s2 = e1.state(), e2.state()
    for k in ("w", "a", "b"):
        assert rel(s1[k], s2[k]) < 1e-5


@pytest.mark.parametrize("F,K,beta,iters,N,restart", [
    (4097, 8, 64, 3, 256, "warm"),   # 8192-point STFT rows: W does not fit shared memory (generic kernel)
    (65, 300, 64, 2, 128, "fresh"),  # K beyond the tensor-pipe kernel's 256
])
def test_extreme_shapes(F, K, beta, iters, N, restart):
    eng, orc, v = make_pair(F, K, beta, iters, N, restart=restart, rho=0.8)
    orc.run(v.astype(np.float64))
    eng.run(v)
    se, so = eng.state(), orc.state()
    for k in ("w", "a", "b"):
        assert rel(se[k], so[k]) < RTOL, (k, rel(se[k], so[k]))
    assert se["commits"] == so["commits"]
