"""Where the config-3 e2e step goes: state init, the host-frame pass (chunked H2D + compute),
the dictionary read back.  Host wall clock with a device synchronize after each part."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1106_4198_b200 as E  # noqa: E402
from tools.synth import spectrogram_torch, w_init  # noqa: E402

F, K, beta, iters, N = 513, 50, 4096, 10, 2_700_000
vd = spectrogram_torch(F, K, N, seed=1)
vh = torch.empty_like(vd, device="cpu").pin_memory()
vh.copy_(vd)
del vd
torch.cuda.empty_cache()
eng = E.Online(F, K, beta, iters, restart="warm", n_store=N)
w0 = w_init(F, K, 2)
a0 = np.full((F, K), 1e-3)
wbuf = np.empty((F, K), order="F")
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.set_dictionary(w0, a0, a0)
    eng.set_counters(0, 0, 0.95967)
    t1 = time.perf_counter()
    eng.fill_warm_h(1.0)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    eng.enqueue(vh, N, vh.stride(0))
    t3 = time.perf_counter()
    eng.synchronize()
    t4 = time.perf_counter()
    E.lib().isnmf_online_get_dictionary(eng._h, E._p(wbuf), None, None)
    t5 = time.perf_counter()
    print(f"set W/A/B + counters {1e3*(t1-t0):.2f} ms | fill_warm_h (synced) {1e3*(t2-t1):.2f} | enqueue returns {1e3*(t3-t2):.2f} | "
          f"pass done {1e3*(t4-t2):.2f} ({N*F*4/(t4-t2)/1e9:.1f} GB/s) | read back {1e3*(t5-t4):.2f} | total {1e3*(t5-t0):.2f} ms", flush=True)
