"""Per-phase cycle breakdown of K1 (needs `make prof`: lib_prof/ build)."""
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
F, K, beta, iters = 513, 50, 4096, 10
N = beta * 20
vd = spectrogram_torch(F, K, N, seed=1)
torch.cuda.synchronize()
eng = E.Online(F, K, beta, iters, restart="warm", n_store=N)
eng.set_dictionary(w_init(F, K, 2), np.full((F, K), 1e-3), np.full((F, K), 1e-3))
eng.set_counters(0, 0, 0.96)
eng.fill_warm_h(1.0)
L.isnmf_debug_phase_prof(eng._h, None, 0, 1)
eng.enqueue(vd, N, vd.stride(0))
eng.synchronize()
nblk = (beta + 27) // 28
buf = np.zeros(nblk * 8 * 8, dtype=np.int64)
L.isnmf_debug_phase_prof(eng._h, buf.ctypes.data_as(C.c_void_p), buf.size, 1)
b = buf.reshape(nblk, 8, 8) / 20.0  # per launch
names = ["prologue", "phaseA", "phaseB", "barrier-wait", "partials+update", "stats-phaseA+div", "stats", "epilogue"]
tot = b.sum(axis=2)
print("cycles per launch per warp: mean %.0f max %.0f" % (tot.mean(), tot.max()))
for i, n in enumerate(names):
    col = b[:, :, i]
    print(f"{n:18s} mean {col.mean():9.0f}  ({100 * col.mean() / tot.mean():5.1f}%)  min {col.min():9.0f} max {col.max():9.0f}")
print("per-warp total (CTA 0):", tot[0].astype(int))
