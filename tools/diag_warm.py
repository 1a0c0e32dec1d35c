"""Diagnose long warm runs at config 3: per pass, the distribution of the
stored activations (min, zeros, count below thresholds) and where the first
failure happens.  Usage: python tools/diag_warm.py [passes]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1106_4198_b200 as E  # noqa: E402
from tools.synth import CONFIGS, spectrogram_torch, w_init  # noqa: E402

passes = int(sys.argv[1]) if len(sys.argv) > 1 else 26
cfg = CONFIGS["c3"]
F, K, beta, iters, N, rho = cfg["F"], cfg["K"], cfg["beta"], cfg["iters"], cfg["N"], cfg["rho"]
torch.cuda.set_device(0)
vd = spectrogram_torch(F, K, N, seed=1000, shape=cfg["shape"], device="cuda")
w0 = w_init(F, K, 77)
a0 = np.full((F, K), 1e-3)
eng = E.Online(F, K, beta, iters, restart="warm", n_store=N)
eng.set_dictionary(w0, a0, a0)
eng.set_counters(0, 0, rho)
eng.fill_warm_h(1.0)
for p in range(passes):
    t0 = time.time()
    try:
        eng.run(vd)
    except E.EngineError as e:
        print(f"pass {p}: FAILED {e}", flush=True)
        break
    st = eng.state(warm_h=True)
    h = st["warm_h"]
    pos = h[h > 0]
    print(f"pass {p}: t={st['t']} commits={st['commits']} obj={st['last_minibatch_obj']:.6g} "
          f"min={h.min():.3e} min_pos={pos.min() if pos.size else 0:.3e} zeros={int((h <= 0).sum())} "
          f"nan={int(np.isnan(h).sum())} <1e-30={int((h < 1e-30).sum())} <1e-20={int((h < 1e-20).sum())} "
          f"<1e-10={int((h < 1e-10).sum())} max={h.max():.3e} w_min={st['w'].min():.3e} "
          f"a_min={st['a'].min():.3e} b_min={st['b'].min():.3e} ({time.time() - t0:.1f}s)", flush=True)
