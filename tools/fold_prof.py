"""Per-phase globaltimer stamps of the last K2 (fold_commit_kernel) launch (needs `make prof`)."""
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
L.isnmf_debug_fold_prof.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
F, K, beta, iters = 513, 50, 4096, 10
N = beta * 20
vd = spectrogram_torch(F, K, N, seed=1)
torch.cuda.synchronize()
eng = E.Online(F, K, beta, iters, restart="warm", n_store=N)
eng.set_dictionary(w_init(F, K, 2), np.full((F, K), 1e-3), np.full((F, K), 1e-3))
eng.set_counters(0, 0, 0.96)
eng.fill_warm_h(1.0)
L.isnmf_debug_fold_prof(eng._h, None, 0)
eng.enqueue(vd, N, vd.stride(0))
eng.synchronize()
buf = np.zeros(K * 4 * 8, dtype=np.int64)
L.isnmf_debug_fold_prof(eng._h, buf.ctypes.data_as(C.c_void_p), buf.size)
b = buf.reshape(K * 4, 8).astype(np.float64)
t0 = b[:, 0].min()
names = ["start", "phase1 loads", "cluster sync 1", "pending/commit rows", "cs sync", "rescale rows", "ticket", "last CTA end"]
for i, n in enumerate(names):
    col = b[:, i]
    col = col[col > 0]
    if len(col) == 0:
        continue
    r = (col - t0) / 1e3
    print(f"{n:22s} us from first start: min {r.min():7.2f} median {np.median(r):7.2f} max {r.max():7.2f}")
