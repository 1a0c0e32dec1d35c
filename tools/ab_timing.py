"""A/B wall time of the online path for several builds of the engine, in one
process each (usage: ab_timing.py N lib1.so [lib2.so ...]); prints frames/s."""
import subprocess
import sys

N = sys.argv[1]
code = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_1106_4198_b200 as E
E.LIB_PATH = sys.argv[2]
from tools.synth import spectrogram_torch, w_init
F, K, beta, iters = 513, 50, 4096, 10
N = int(sys.argv[1])
vd = spectrogram_torch(F, K, N, seed=1); torch.cuda.synchronize()
eng = E.Online(F, K, beta, iters, restart="warm", n_store=N)
eng.set_dictionary(w_init(F, K, 2), np.full((F, K), 1e-3), np.full((F, K), 1e-3))
eng.set_counters(0, 0, 0.96); eng.fill_warm_h(1.0)
best = 0
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    eng.enqueue(vd, N, vd.stride(0)); eng.synchronize()
    best = max(best, N / (time.perf_counter() - t0))
print(f"{sys.argv[2]}: {best:.4e} frames/s")
'''
for lib in sys.argv[2:] * 2:
    r = subprocess.run([sys.executable, "-c", code, N, lib], capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-500:])
