"""Free-running config-3 trajectory on the device against the fp64 oracle (the
oracle is pinned to the reference's own trainers by test_oracle_ref_trainers.py).

Config 3's shape and state (F=513, K=50, beta=4096, I=10, rho = 0.99^(4096/1000),
W0 ~ U(0.1, 1) l1-normalised, A0 = B0 = 1e-3, warm store H0 = 1) over 49,152
frames visited twice: 24 consecutive mini-batches, the second pass warm-started
from activations stored and rescaled by every commit since (the P-table path,
model.hpp:84).  Per-commit mini-batch objective, final W, A, B and every stored
activation within the north-star 1e-4 relative.
"""
import numpy as np
import pytest

import oracle as O
import paper_1106_4198_b200 as E
from tools.synth import CONFIGS, spectrogram_np, w_init

pytestmark = pytest.mark.gpu
RTOL = 1e-4


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def test_c3_free_running_24_minibatches_two_passes():
    import torch
    c = CONFIGS["c3"]
    F, K, beta, iters, rho = c["F"], c["K"], c["beta"], c["iters"], c["rho"]
    N, passes = 12 * beta, 2
    v = spectrogram_np(F, K, N, seed=3131)
    w0 = w_init(F, K, 3132)
    a0 = np.full((F, K), 1e-3)

    eng = E.Online(F, K, beta, iters, restart="warm", n_store=N)
    eng.set_dictionary(w0, a0, a0)
    eng.set_counters(0, 0, rho)
    eng.fill_warm_h(1.0)
    vd = torch.from_numpy(np.ascontiguousarray(v.T)).cuda()
    for _ in range(passes):
        eng.run(vd)
    se = eng.state(warm_h=True)
    ts, to, _ = eng.trace()
    eng.close()

    orc = O.Online(w0, beta=beta, r=1.0, inner_iters=iters, restart="warm", dataset_size=N,
                   dataset=v.astype(np.float64))
    orc.set(a=a0, b=a0, rho=rho, t=0, commits=0, warm_h=np.ones((K, N)))
    tt, tobj = [], []
    for _ in range(passes):
        t1, o1 = orc.run(v.astype(np.float64))
        tt.append(t1)
        tobj.append(o1)
    so = orc.state(warm_h=True)
    tt, tobj = np.concatenate(tt), np.concatenate(tobj)

    assert se["commits"] == so["commits"] == 24
    np.testing.assert_array_equal(ts, tt)
    assert rel(to, tobj) < RTOL, rel(to, tobj)
    for k in ("w", "a", "b", "warm_h"):
        assert rel(se[k], so[k]) < RTOL, (k, rel(se[k], so[k]))
    assert rel(se["last_delta"], so["last_delta"]) < 1e-3  # ||dW||_F of nearby dictionaries
