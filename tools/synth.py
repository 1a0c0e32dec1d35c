"""Seeded synthetic power spectrograms for the BASELINE.json configs.

V = (W* H*) .* E + 1e-9 in fp32 (configs 0-4): W* ~ U(0.1, 1) with unit-l1
columns, H* ~ Gamma(shape, 1) (0.5; 0.3 for the large-K config), E ~ Exp(1)
(the multiplicative noise of a complex-Gaussian STFT power).  The paper's
audio is proprietary; these stand in for it with the shapes and
value distributions BASELINE.json names.  Initial state: W0 ~ U(0.1, 1),
l1-normalised (online.hpp:263 requires it), A0 = B0 = 1e-3, H0 = 1.
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    # name: (F, K, beta, inner_iters, N, rho, gamma_shape)
    "c0": dict(F=257, K=10, beta=100, iters=5, N=10_000, rho=1.0, shape=0.5),
    "c1": dict(F=513, K=20, beta=1000, iters=10, N=225_000, rho=1.0, shape=0.5),
    "c2": dict(F=513, K=50, beta=None, iters=1, N=225_000, rho=None, shape=0.5, epochs=100),
    "c3": dict(F=513, K=50, beta=4096, iters=10, N=2_700_000, rho=0.99 ** (4096 / 1000), shape=0.5),
    "c4": dict(F=1025, K=256, beta=8192, iters=8, N=500_000, rho=1.0, shape=0.3),
}


def w_init(F, K, seed):
    rng = np.random.default_rng(seed)
    w = rng.uniform(0.1, 1.0, size=(F, K))
    return np.asfortranarray(w / w.sum(axis=0, keepdims=True))


def spectrogram_np(F, K, N, seed, shape=0.5):
    """Host generator (tests, small N): returns V as F x N fp32 column-major."""
    rng = np.random.default_rng(seed)
    ws = rng.uniform(0.1, 1.0, size=(F, K))
    ws /= ws.sum(axis=0, keepdims=True)
    hs = rng.gamma(shape, 1.0, size=(K, N))
    e = rng.exponential(1.0, size=(F, N))
    v = (ws @ hs) * e + 1e-9
    return np.asfortranarray(v.astype(np.float32))


def spectrogram_torch(F, K, N, seed, shape=0.5, device="cuda", ld=None):
    """Device generator (bench, large N): returns a torch tensor [N, ld] fp32
    (row n = frame n, F valid entries) generated in blocks on `device`."""
    import torch
    ld = ld or F
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    ws = torch.rand(F, K, generator=g, device=device, dtype=torch.float64) * 0.9 + 0.1
    ws /= ws.sum(dim=0, keepdim=True)
    ws32 = ws.float()
    out = torch.empty(N, ld, device=device, dtype=torch.float32)
    blk = 1 << 18
    for s in range(0, N, blk):
        n = min(blk, N - s)
        conc = torch.full((n, K), shape, device=device, dtype=torch.float32)
        hs = torch._standard_gamma(conc, generator=g)
        e = torch.empty(n, F, device=device, dtype=torch.float32).exponential_(1.0, generator=g)
        out[s:s + n, :F] = (hs @ ws32.T) * e + 1e-9
    if ld > F:
        out[:, F:] = 0
    return out

