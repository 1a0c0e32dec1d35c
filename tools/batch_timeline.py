"""Timeline of the batch path's K1M (multi-tile) in CTA 0 (needs `make prof`): cycles of the
last frame tile the CTA ran — H0 set-up, the MM pass (chunk MMAs / barrier / update / barrier),
statistics preparation, statistics blocks, final h.  usage: batch_timeline.py [epochs]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1106_4198_b200 as E  # noqa: E402

E.LIB_PATH = os.path.join(os.path.dirname(E.LIB_PATH), "..", "lib_prof", "libisnmf_b200.so")
from tools.synth import spectrogram_torch  # noqa: E402

L = E.lib()
L.isnmf_debug_work_prof.argtypes = [C.c_void_p, C.c_int64]
epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 3
F, K, N = 513, 50, 225_000
vd = spectrogram_torch(F, K, N, seed=7, device="cuda")
rng = np.random.default_rng(8)
w0 = rng.uniform(0.1, 1.0, size=(F, K))
h0 = rng.uniform(0.1, 1.0, size=(K, N))
L.isnmf_debug_work_prof(None, 0)
E.batch_profile(1)
out = E.batch_train(vd, w0, h0, epochs)
ms, n = E.batch_profile()
print(f"epochs {out['epochs']} device {ms:.3f} ms ({ms / max(1, epochs):.3f} ms/epoch incl. final pass) launches {n}")
nw = 12
buf = np.zeros(16 * 64, dtype=np.int64)
L.isnmf_debug_work_prof(buf.ctypes.data_as(C.c_void_p), buf.size)
ts = buf[: nw * 64].reshape(nw, 64)
t0 = ts[:, 59].min()
print("cycles from the tile start (stamp 59) per warp:")
print("warp  h0-ready  chunks  bar1  update  bar2  stats-prep  stats-end(61)  blocks: phaseA'/qr/mma/stores")
for w in range(nw):
    r = ts[w]
    blocks = []
    for j in range(4):
        e = 44 + 4 * j
        if r[e] <= r[59] or e + 3 >= 60:
            break
        end = r[e + 4] if (e + 4 < 60 and r[e + 4] > r[e]) else r[61]
        blocks.append(f"{r[e + 1] - r[e]}/{r[e + 2] - r[e + 1]}/{r[e + 3] - r[e + 2]}/{end - r[e + 3]}")
    print(f"{w:3d} {r[0] - t0:8d} {r[1] - r[0]:7d} {r[2] - r[1]:6d} {r[3] - r[2]:6d} {r[4] - r[3]:6d} "
          f"{r[44] - r[60]:8d} {r[61] - t0:10d}    " + "  ".join(blocks))
print(f"kernel: entry -> exit {ts[:, 63].max() - ts[:, 62].min()} cycles (all tiles of CTA 0)")
