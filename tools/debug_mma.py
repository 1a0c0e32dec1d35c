"""K1M debugging aid: repeated solve_h / evaluate_heldout at small shapes (bitwise run-to-run check)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1106_4198_b200 as E  # noqa: E402
from tools.synth import spectrogram_np, w_init  # noqa: E402

for F, K, N in [(33, 3, 40), (33, 3, 2000)]:
    v = spectrogram_np(F, K, N, seed=41)
    v[:, ::7] = 1e-9
    v = v.astype(np.float32)
    w = w_init(F, K, seed=42)
    ds = [E.evaluate_heldout(v, w, 1e-12, 100) for _ in range(4)]
    print("heldout", F, K, N, ds, flush=True)
    hs = [E.solve_h(v.astype(np.float64), w, np.ones((K, N)), 20, 1e-12) for _ in range(4)]
    print("solve_h equal:", [bool(np.array_equal(hs[0], h)) for h in hs], float(np.max(hs[0])), flush=True)
    big = [np.zeros(1 << 26, np.float32) + i for i in range(2)]  # churn the allocator
    ds = [E.evaluate_heldout(v, w, 1e-12, 100) for _ in range(2)]
    print("heldout after churn", ds, flush=True)
