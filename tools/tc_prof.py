"""Window timeline of K1T at config 4 (clock64 stamps of CTA 0, pass 1; needs `make prof`)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1106_4198_b200 as E  # noqa: E402

E.LIB_PATH = os.path.join(os.path.dirname(E.LIB_PATH), "..", "lib_prof", "libisnmf_b200.so")
from tools.synth import spectrogram_torch, w_init  # noqa: E402

L = E.lib()
L.isnmf_debug_phase_prof.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32]
F, K, beta, iters = 1025, 256, 8192, 8
N = beta * 2
vd = spectrogram_torch(F, K, N, seed=1)
torch.cuda.synchronize()
eng = E.Online(F, K, beta, iters, restart="warm", n_store=N)
eng.set_dictionary(w_init(F, K, 2), np.full((F, K), 1e-3), np.full((F, K), 1e-3))
eng.set_counters(0, 0, 1.0)
eng.fill_warm_h(1.0)
L.isnmf_debug_phase_prof(eng._h, None, 0, 1)
eng.enqueue(vd, N, vd.stride(0))
eng.synchronize()
buf = np.zeros(40 * 8, dtype=np.int64)
L.isnmf_debug_phase_prof(eng._h, buf.ctypes.data_as(C.c_void_p), buf.size, 0)
b = buf.reshape(40, 8)[:33].astype(np.int64)
print("window: issue(tid0)  phaseA(w1)  wait  epilogue  stage_w  barrier  (cycles from the window start, warp 1)")
for w, r in enumerate(b[:8]):
    print(w, [int(r[i] - r[0]) if r[i] else None for i in range(1, 7)])
print("window period:", np.diff(b[:, 0]).tolist())
