"""Timing probe of the online path (device-resident frames)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1106_4198_b200 as E  # noqa: E402
from tools.synth import spectrogram_torch, w_init  # noqa: E402

F, K, beta, iters = 513, 50, 4096, 10
N = int(sys.argv[1]) if len(sys.argv) > 1 else 409600
vd = spectrogram_torch(F, K, N, seed=1)
torch.cuda.synchronize()
eng = E.Online(F, K, beta, iters, restart="warm", n_store=N)
eng.set_dictionary(w_init(F, K, 2), np.full((F, K), 1e-3), np.full((F, K), 1e-3))
eng.set_counters(0, 0, 0.96)
eng.fill_warm_h(1.0)
for rep in range(4):
    prof = E.Profile(eng)
    prof.start()
    t0 = time.perf_counter()
    eng.enqueue(vd, N, vd.stride(0))
    t1 = time.perf_counter()
    eng.synchronize()
    t2 = time.perf_counter()
    k = prof.stop()
    print(f"rep {rep}: enqueue {1e3*(t1-t0):.2f} ms, sync {1e3*(t2-t1):.2f} ms, span {k['span_ms']:.2f} ms, "
          f"k1 {k['solve_ms']:.2f} ms / {k['solve_launches']} launches, k2+k3 {k['tail_ms']:.2f} ms, "
          f"frames/s {N/(k['span_ms']/1e3):.3e}")
# without per-kernel events: wall time of enqueue+synchronize
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.enqueue(vd, N, vd.stride(0))
    eng.synchronize()
    t2 = time.perf_counter()
    print(f"no-events rep {rep}: wall {1e3*(t2-t0):.2f} ms, frames/s {N/(t2-t0):.3e}")
