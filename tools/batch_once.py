"""One batch_train call at the config-2 shape (F=513, K=50, N=225k) with a few
epochs, for launch lists / ncu captures of the batch path.
usage: python tools/batch_once.py [epochs]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1106_4198_b200 as E  # noqa: E402
from tools.synth import spectrogram_torch  # noqa: E402

epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 3
F, K, N = 513, 50, 225_000
vd = spectrogram_torch(F, K, N, seed=7, device="cuda")
rng = np.random.default_rng(8)
w0 = rng.uniform(0.1, 1.0, size=(F, K))
h0 = rng.uniform(0.1, 1.0, size=(K, N))
E.batch_profile(1)
out = E.batch_train(vd, w0, h0, epochs)
ms, n = E.batch_profile()
print(f"epochs {out['epochs']} device {ms:.3f} ms ({ms / max(1, epochs):.3f} ms/epoch incl. final pass) launches {n}")
