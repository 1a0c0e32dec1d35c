"""K1 time per launch at arbitrary (F, K, beta, iters) with device-resident frames
(A/B aid: e.g. the cost of F's tail rows).  usage: k1_time.py F K beta iters [F K beta iters ...]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1106_4198_b200 as E  # noqa: E402
from tools.synth import spectrogram_torch, w_init  # noqa: E402

args = [int(x) for x in sys.argv[1:]]
for i in range(0, len(args), 4):
    F, K, beta, iters = args[i:i + 4]
    N = beta * 40
    vd = spectrogram_torch(F, K, N, seed=1)
    torch.cuda.synchronize()
    eng = E.Online(F, K, beta, iters, restart="warm", n_store=N)
    eng.set_dictionary(w_init(F, K, 2), np.full((F, K), 1e-3), np.full((F, K), 1e-3))
    eng.set_counters(0, 0, 0.96)
    eng.fill_warm_h(1.0)
    eng.run(vd[: beta * 4], beta * 4, vd.stride(0))
    p = E.Profile(eng, per_kernel=True)
    p.start()
    eng.run(vd, N, vd.stride(0))
    s = p.stop()
    print(f"F={F} K={K} beta={beta} I={iters}: K1 {1e3 * s['solve_ms'] / s['solve_launches']:.1f} us/launch, "
          f"step {1e3 * s['span_ms'] / (N / beta):.1f} us/minibatch", flush=True)
    eng.close()
