"""Host wall clock of batch_train calls at the config-2 shape with V in pinned host memory,
five calls in a row (the e2e leg of the c2 bench line varies with host page faults)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1106_4198_b200 as E  # noqa: E402
from tools.synth import spectrogram_torch  # noqa: E402

F, K, N, epochs = 513, 50, 225_000, int(sys.argv[1]) if len(sys.argv) > 1 else 100
vd = spectrogram_torch(F, K, N, seed=7, device="cuda")
vh = torch.empty_like(vd, device="cpu").pin_memory()
vh.copy_(vd)
del vd
rng = np.random.default_rng(8)
w0 = rng.uniform(0.1, 1.0, size=(F, K))
h0 = np.asfortranarray(rng.uniform(0.1, 1.0, size=(K, N)))
E.batch_profile(1)
for i in range(5):
    t0 = time.perf_counter()
    out = E.batch_train(vh, w0, h0, epochs)
    t1 = time.perf_counter()
    ms, n = E.batch_profile()
    print(f"call {i}: wall {1e3 * (t1 - t0):.1f} ms, device {ms:.1f} ms, overhead {1e3 * (t1 - t0) - ms:.1f} ms", flush=True)
