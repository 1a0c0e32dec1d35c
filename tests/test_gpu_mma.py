"""Parity of K1M (csrc/kernels_mma.cuh, the all-tensor-pipe solve for K <= 56)
at the shapes that exercise its edges, and of the kernels it replaced.

* one frame group (<= 16 frames per CTA) and two (17..32), a partly filled
  frame group (17 frames), K a multiple of 8 (no padded k) and K = 1;
* F not a multiple of 8 or 16 (padded dictionary rows), F so large that the
  12-warp CTA does not fit shared memory (the 8-warp fallback);
* the FFMA register-tile kernels (ISNMF_MMA=0) and the 8-warp K1M
  (ISNMF_MMA_WARPS=8) against the oracle, in subprocesses (the switches are read
  once per process).
Each case is one mini-batch from an injected state (test_gpu_online's
protocol): W, A, B, warm H and the mini-batch objective within 1e-4 relative.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
import paper_1106_4198_b200 as E
from tools.synth import spectrogram_np, w_init

pytestmark = pytest.mark.gpu
RTOL = 1e-4
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def one_minibatch(F, K, beta, iters, restart="warm", seed=5):
    rng = np.random.default_rng(F * 7 + K)
    v = spectrogram_np(F, K, beta, seed=seed + 1)
    w = w_init(F, K, seed=seed)
    a = rng.uniform(0.5, 2.0, size=(F, K)) * w * w
    b = rng.uniform(0.5, 2.0, size=(F, K))
    eng = E.Online(F, K, beta, iters, restart=restart, seed=seed, n_store=beta if restart == "warm" else 0)
    eng.set_dictionary(w, a, b)
    eng.set_counters(0, 0, 0.9)
    orc = O.Online(w, beta=beta, r=1.0, inner_iters=iters, restart=restart, seed=seed, dataset_size=beta,
                   dataset=v.astype(np.float64) if restart == "warm" else None)
    orc.set(a=a, b=b, rho=0.9, t=0, commits=0)
    if restart == "warm":
        h0 = rng.gamma(2.0, 0.5, size=(K, beta)) + 1e-2
        eng.set_warm_h(h0)
        orc.set(warm_h=h0, rho=0.9, t=0, commits=0)
    orc.run(v.astype(np.float64))
    eng.run(v)
    so = orc.state(warm_h=restart == "warm")
    se = eng.state(warm_h=restart == "warm")
    errs = {k: rel(se[k], so[k]) for k in ("w", "a", "b")}
    errs["obj"] = rel(se["last_minibatch_obj"], so["last_minibatch_obj"])
    if restart == "warm":
        errs["warm_h"] = rel(se["warm_h"], so["warm_h"])
    assert se["commits"] == so["commits"] == 1
    return errs


@pytest.mark.parametrize("F,K,beta,iters,restart", [
    (100, 56, 600, 6, "warm"),     # K = 56: no padded k; 5 frames per CTA (one frame group)
    (513, 50, 2368, 4, "warm"),    # 16 frames per CTA: one full frame group
    (513, 50, 2516, 4, "fresh"),   # 17 frames per CTA: second frame group holds one frame
    (33, 8, 4736, 5, "warm"),      # KB = 1, F = 33 (rows padded to 48), 32 frames per CTA
    (257, 1, 1000, 5, "warm"),     # K = 1
    (600, 50, 4096, 3, "warm"),    # 12-warp CTA does not fit: 8-warp fallback
])
def test_k1m_edge_shapes(F, K, beta, iters, restart):
    errs = one_minibatch(F, K, beta, iters, restart)
    assert max(errs.values()) < RTOL, errs


SNIPPET = """
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + '/oracle'); sys.path.insert(0, {root!r} + '/tests')
from test_gpu_mma import one_minibatch
for shape in [(513, 50, 4096, 10, 'warm'), (257, 10, 100, 5, 'fresh'), (513, 20, 1000, 10, 'warm')]:
    e = one_minibatch(*shape)
    print(shape, max(e.values()))
    assert max(e.values()) < 1e-4, e
print('variant ok')
"""


@pytest.mark.parametrize("env", [{"ISNMF_MMA": "0"}, {"ISNMF_MMA_WARPS": "8"}])
def test_solve_variants_subprocess(env):
    r = subprocess.run([sys.executable, "-c", SNIPPET.format(root=ROOT)], capture_output=True, text=True,
                       timeout=600, env={**os.environ, **env}, cwd=ROOT)
    assert r.returncode == 0 and "variant ok" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
