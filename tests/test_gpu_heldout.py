"""evaluate_heldout (harness.hpp:17-37) on the device against the fp64 oracle.

The random init is the reference's stream (pinned on CPU in
test_oracle_trainers.py); the MM iterations and the final divergence run in the
fused solve kernel at frozen W.  Tolerance: 1e-4 relative (north_star).
"""
import numpy as np
import pytest

import oracle as O
import paper_1106_4198_b200 as E
from tools.synth import spectrogram_np, w_init

pytestmark = pytest.mark.gpu
RTOL = 1e-4


@pytest.mark.parametrize("F,K,N,iters,seed", [
    (65, 4, 50, 100, 0x45),    # reference defaults (100 iterations, seed 0x45)
    (513, 50, 300, 100, 0x45),  # config-3 dictionary shape
    (129, 8, 77, 0, 3),         # no iterations: divergence of the random init
    (33, 3, 20000, 10, 11),     # several launch segments
    (1025, 256, 64, 8, 5),      # config-4 shape (generic kernel)
])
def test_heldout_matches_oracle(F, K, N, iters, seed):
    v = spectrogram_np(F, K, N, seed=F + N).astype(np.float32)
    w = w_init(F, K, seed=7)
    dev = E.evaluate_heldout(v, w, 1e-12, iters, seed)
    ref = O.evaluate_heldout(w, v.astype(np.float64), 1e-12, iters, seed)
    assert abs(dev - ref) <= RTOL * abs(ref), (dev, ref)


def test_heldout_device_frames_and_errors():
    import torch
    F, K, N = 65, 5, 120
    v = spectrogram_np(F, K, N, seed=1).astype(np.float32)
    w = w_init(F, K, seed=2)
    host = E.evaluate_heldout(v, w)
    dev = E.evaluate_heldout(torch.from_numpy(np.ascontiguousarray(v.T)).cuda(), w)
    assert host == dev
    with pytest.raises(E.EngineError) as e:
        E.evaluate_heldout(v[:, :0], w)
    assert e.value.kind == "EmptyDataset"
