"""Host-side enqueue cost per mini-batch (tiny F/K so GPU work is negligible)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1106_4198_b200 as E  # noqa: E402

for (F, K, beta) in [(16, 4, 64), (513, 50, 4096)]:
    N = beta * 400
    vd = torch.rand(N, F, device="cuda") + 0.1
    eng = E.Online(F, K, beta, 1, restart="warm", n_store=N)
    w = np.full((F, K), 1.0 / F)
    eng.set_dictionary(w, w * w, np.ones((F, K)))
    eng.fill_warm_h(1.0)
    eng.enqueue(vd, N, vd.stride(0))
    eng.synchronize()
    for rep in range(2):
        t0 = time.perf_counter()
        eng.enqueue(vd, N, vd.stride(0))
        t1 = time.perf_counter()
        eng.synchronize()
        t2 = time.perf_counter()
        print(f"F={F} K={K} beta={beta}: {400} mini-batches enqueue {1e3*(t1-t0):.1f} ms "
              f"({1e6*(t1-t0)/400:.1f} us/mb), total {1e3*(t2-t0):.1f} ms")
