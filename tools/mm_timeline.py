"""Timeline of K1M in CTA 0 (needs `make prof`): per warp and pass, cycles in the
chunk MMAs, waiting at the group barrier, the reduction/update and its barrier."""
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
F, K, beta, iters = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (513, 50, 4096, 10)
N = beta * 3
vd = spectrogram_torch(F, K, N, seed=1)
torch.cuda.synchronize()
eng = E.Online(F, K, beta, iters, restart="warm", n_store=N)
eng.set_dictionary(w_init(F, K, 2), np.full((F, K), 1e-3), np.full((F, K), 1e-3))
eng.set_counters(0, 0, 0.96)
eng.fill_warm_h(1.0)
L.isnmf_debug_phase_prof(eng._h, None, 0, 1)
eng.enqueue(vd, N, vd.stride(0))
eng.synchronize()
nw = 12
buf = np.zeros(4096, dtype=np.int64)
L.isnmf_debug_phase_prof(eng._h, buf.ctypes.data_as(C.c_void_p), buf.size, 0)
ts = buf[: nw * 64].reshape(nw, 64).astype(np.int64)
t0 = ts[:, 62].min()
print("warp  prologue  " + "  ".join(f"p{p}:mma/bar1/upd/bar2" for p in range(3)) + "  ...  stats  total")
tot = np.zeros(4)
for w in range(nw):
    r = ts[w]
    parts = []
    prev = r[0]
    for p in range(iters):
        e = [r[1 + 4 * p], r[2 + 4 * p], r[3 + 4 * p], r[4 + 4 * p]]
        d = [e[0] - prev, e[1] - e[0], e[2] - e[1], e[3] - e[2]]
        tot += d
        parts.append("/".join(str(int(x)) for x in d))
        prev = e[3]
    print(f"{w:3d} {r[0] - t0:8d}  " + "  ".join(parts[:3]) + f"  ...  {r[61] - r[60]:6d}  {r[61] - t0:7d}")
tot /= nw * iters
print("per pass (mean over warps / max over warps): mma, bar1, update, bar2")
for p in range(iters):
    prev = ts[:, 4 * p] if p else ts[:, 0]
    e = [ts[:, 1 + 4 * p], ts[:, 2 + 4 * p], ts[:, 3 + 4 * p], ts[:, 4 + 4 * p]]
    d = [e[0] - prev, e[1] - e[0], e[2] - e[1], e[3] - e[2]]
    print(f"  pass {p}: " + "  ".join(f"{int(x.mean())}/{int(x.max())}" for x in d) + f"   pass total {int((e[3] - prev).max())}")
print("mean per pass: mma %.0f  bar1 %.0f  update %.0f  bar2 %.0f" % tuple(tot))
print("statistics blocks (cycles): phaseA' / q,r,div / stats MMAs / stores")
for w in range(nw):
    r = ts[w]
    out = []
    for j in range(4):
        e = 44 + 4 * j
        if r[e] == 0 or e + 3 >= 60:
            break
        end = r[e + 4] if (e + 4 < 60 and r[e + 4] > r[e]) else r[61]
        out.append(f"{r[e + 1] - r[e]}/{r[e + 2] - r[e + 1]}/{r[e + 3] - r[e + 2]}/{end - r[e + 3]}")
    print(f"{w:3d}  " + "  ".join(out) + f"   (prep {r[44] - r[60]})")
print("absolute stamps (cycles from CTA start) of passes 3-4: chunks-done / update-start / update-end")
for w in range(nw):
    r = ts[w]
    print(f"{w:3d} grp{int(w >= nw // 2)}  " + "  ".join(f"{r[1 + 4 * p] - t0}/{r[2 + 4 * p] - t0}/{r[3 + 4 * p] - t0}" for p in (3, 4)))
print("prologue (entry -> passes) / stats end -> exit, cycles:")
for w in range(nw):
    r = ts[w]
    print(f"{w:3d}  entry {r[62] - t0:7d}  pdl wait {r[58] - r[62]:6d}  prologue {r[0] - r[58]:6d}  "
          f"stats prep {r[44] - r[60]:6d}  epilogue {r[63] - r[61]:6d}  exit {r[63] - t0:7d}")
