"""Full-size runs of the BASELINE online configs on the device (config 3: 2.7M frames,
config 4: 500k frames at K = 256), held to size-independent properties — the fp64
oracle cannot replay millions of frames inside a test:

* counters and trace: commits = floor(N / beta), the leftover frames pending, one trace
  point per commit at t = 4096 (i + 1), finite positive mini-batch objectives that fall
  from the first mini-batches to the last;
* dictionary invariants after the last commit: W > 0 with unit-l1 columns (the
  rescale of model.hpp:73-86), A, B > 0, everything finite;
* bitwise reproducibility of the whole run (fixed-order reductions);
* parity at a late state: the dictionary, A and B the full run ends with are injected
  into the engine and the oracle, and one more mini-batch (fresh restarts, forgetting
  factor of config 3) is compared at the north-star 1e-4.
"""
import numpy as np
import pytest

import oracle as O
import paper_1106_4198_b200 as E
from tools.synth import CONFIGS, spectrogram_np, spectrogram_torch, w_init

pytestmark = pytest.mark.gpu
RTOL = 1e-4


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def full_run(name, vd):
    import torch
    c = CONFIGS[name]
    F, K, beta, iters, N = c["F"], c["K"], c["beta"], c["iters"], c["N"]
    eng = E.Online(F, K, beta, iters, restart="warm", n_store=N)
    eng.set_dictionary(w_init(F, K, 77), np.full((F, K), 1e-3), np.full((F, K), 1e-3))
    eng.set_counters(0, 0, c["rho"])
    eng.fill_warm_h(1.0)
    eng.run(vd, N, vd.stride(0))
    torch.cuda.synchronize()
    st = eng.state()
    tr = eng.trace()
    eng.close()
    return st, tr


@pytest.fixture(scope="module")
def c3():
    import torch
    c = CONFIGS["c3"]
    vd = spectrogram_torch(c["F"], c["K"], c["N"], seed=1000, shape=c["shape"])
    torch.cuda.synchronize()
    runs = [full_run("c3", vd), full_run("c3", vd)]
    del vd
    torch.cuda.empty_cache()
    return runs


def test_c3_counters_and_trace(c3):
    (st, (s, o, sec)), _ = c3
    c = CONFIGS["c3"]
    commits = c["N"] // c["beta"]
    assert st["commits"] == commits == 659 and st["t"] == c["N"]
    assert st["pending_count"] == c["N"] - commits * c["beta"]
    assert len(s) == commits and np.array_equal(s, c["beta"] * (np.arange(commits, dtype=np.uint64) + 1))
    assert np.all(np.isfinite(o)) and np.all(o > 0)
    assert np.mean(o[-50:]) < np.mean(o[:10])
    assert np.all(np.diff(sec) >= 0)


def test_c3_dictionary_invariants(c3):
    (st, _), _ = c3
    w, a, b = st["w"], st["a"], st["b"]
    for m in (w, a, b):
        assert np.all(np.isfinite(m)) and np.all(m > 0)
    assert np.max(np.abs(w.sum(axis=0) - 1.0)) < 1e-12
    assert np.isfinite(st["last_delta"]) and st["last_delta"] > 0


def test_c3_bitwise_reproducible(c3):
    (s1, t1), (s2, t2) = c3
    for k in ("w", "a", "b", "pending_a", "pending_b"):
        assert np.array_equal(s1[k], s2[k]), k
    assert np.array_equal(t1[1], t2[1])


def test_c3_late_state_parity(c3):
    (st, _), _ = c3
    c = CONFIGS["c3"]
    F, K, beta, iters = c["F"], c["K"], c["beta"], c["iters"]
    v = spectrogram_np(F, K, beta, seed=4242)
    seed, t0, commits = 9, 659 * beta, 659
    eng = E.Online(F, K, beta, iters, restart="fresh", seed=seed)
    eng.set_dictionary(st["w"], st["a"], st["b"])
    eng.set_counters(t0, commits, c["rho"])
    orc = O.Online(st["w"], beta=beta, r=1.0, inner_iters=iters, restart="fresh", seed=seed, dataset_size=beta)
    orc.set(w=st["w"], a=st["a"], b=st["b"], rho=c["rho"], t=t0, commits=commits)
    orc.run(v.astype(np.float64))
    eng.run(v)
    se, so = eng.state(), orc.state()
    for k in ("w", "a", "b"):
        assert rel(se[k], so[k]) < RTOL, (k, rel(se[k], so[k]))
    assert se["commits"] == so["commits"] == commits + 1
    assert rel(se["last_minibatch_obj"], so["last_minibatch_obj"]) < RTOL
    eng.close()


def test_c4_fullsize_properties():
    import torch
    c = CONFIGS["c4"]
    vd = spectrogram_torch(c["F"], c["K"], c["N"], seed=2000, shape=c["shape"])
    torch.cuda.synchronize()
    (s1, (s, o, _)), (s2, _) = full_run("c4", vd), full_run("c4", vd)
    del vd
    torch.cuda.empty_cache()
    commits = c["N"] // c["beta"]
    assert s1["commits"] == commits and s1["pending_count"] == c["N"] - commits * c["beta"]
    assert len(s) == commits and np.all(np.isfinite(o)) and np.all(o > 0)
    assert np.max(np.abs(s1["w"].sum(axis=0) - 1.0)) < 1e-12 and np.all(s1["w"] > 0)
    for k in ("w", "a", "b"):
        assert np.array_equal(s1[k], s2[k]), k
