"""K1 time per launch at the config-3 shape with the frames' leading dimension padded
(ldv = 513 contiguous vs 516 / 520 / 544): the cost of rows that straddle cache lines."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1106_4198_b200 as E  # noqa: E402
from tools.synth import spectrogram_torch, w_init  # noqa: E402

F, K, beta, iters = 513, 50, 4096, 10
N = beta * 40
v0 = spectrogram_torch(F, K, N, seed=1)
for ldv in (513, 516, 520, 544):
    vd = torch.empty(N, ldv, device="cuda", dtype=torch.float32)
    vd[:, :F] = v0
    view = vd[:, :F]
    torch.cuda.synchronize()
    eng = E.Online(F, K, beta, iters, restart="warm", n_store=N)
    eng.set_dictionary(w_init(F, K, 2), np.full((F, K), 1e-3), np.full((F, K), 1e-3))
    eng.set_counters(0, 0, 0.96)
    eng.fill_warm_h(1.0)
    eng.run(view[: beta * 4], beta * 4, ldv)
    p = E.Profile(eng, per_kernel=True)
    p.start()
    eng.run(view, N, ldv)
    s = p.stop()
    print(f"ldv={ldv}: K1 {1e3 * s['solve_ms'] / s['solve_launches']:.1f} us/launch, "
          f"step {1e3 * s['span_ms'] / (N / beta):.1f} us/minibatch", flush=True)
    eng.close()
