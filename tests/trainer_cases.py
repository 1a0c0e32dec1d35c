"""Trainer fixtures produced by the reference itself (tests/golden/gen_trainer_golden.py
runs online_resume / batch_train from /root/reference/proj/include, compiled
unchanged over oracle/ref/eigen_shim) and the runners that replay the same
cases through the fp64 oracle and through the device engine's C ABI."""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
sys.path.insert(0, os.path.join(GOLDEN))
from gen_trainer_golden import BATCH, ONLINE, make_batch_inputs, make_online_inputs  # noqa: E402


def load(name):
    d = np.load(os.path.join(GOLDEN, f"trainer_{name}.npz"))
    return {k: d[k] for k in d.files}


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def check_inputs(fx, v):
    got = hashlib.sha256(np.asfortranarray(v, dtype=np.float32).tobytes(order="F")).hexdigest()
    assert got == str(fx["v_sha256"]), "synthetic V changed since the fixture was generated (numpy version?)"


def chunkstream_order(N, chunks, buffer, seed, budget):
    """Frame order of the reference's ChunkStreamSource (online.hpp:172-210) over the
    columns 0..N-1 sent as chunks of the given sizes (cycled): whole chunks are read
    until `buffer` frames are pending, the first min(buffer, pending) are permuted by
    Fisher-Yates from mt19937_64(mix_seed(seed, block)) and handed out in that order."""
    import oracle as O
    sizes = [int(x) for x in str(chunks).split(",")]
    pending, ready, out = [], [], []
    col, ci, block = 0, 0, 0
    while len(out) < budget:
        if not ready:
            while len(pending) < buffer and col < N:
                cnt = min(sizes[ci % len(sizes)], N - col)
                pending.extend(range(col, col + cnt))
                col += cnt
                ci += 1
            if not pending:
                break
            L = min(buffer, len(pending))
            perm = O.cycle_permutation(seed, block, L)
            block += 1
            ready.extend(pending[int(p)] for p in perm)
            del pending[:L]
        out.append(ready.pop(0))
    return np.asarray(out, dtype=np.uint64)


def visit_order(c):
    """Dataset columns of samples t = 0 .. budget-1 in the case's source order:
    identity (t mod N), the reference's CyclingSource (a fresh Fisher-Yates
    permutation per cycle from mt19937_64(mix_seed(seed, cycle)), online.hpp:79-87)
    or its ChunkStreamSource (chunkstream_order)."""
    import oracle as O
    N, budget = c["N"], c["budget"]
    if c["order"] == "in_order":
        return np.arange(budget, dtype=np.uint64) % np.uint64(N)
    if c["order"] == "chunkstream":
        return chunkstream_order(N, c["chunks"], c["buffer"], c["seed"], budget)
    perms = [O.cycle_permutation(c["seed"], cyc, N) for cyc in range((budget + N - 1) // N)]
    return np.concatenate(perms)[:budget].astype(np.uint64)


def initial_stats(c, w0):
    """A0, B0: BASELINE's a0 fill when the case sets one, else the reference default
    (make_online_state, online.hpp:276-277: delta W0^2 and delta with delta = 1)."""
    if "a0" in c:
        a = np.full(w0.shape, c["a0"])
        return a, a.copy()
    return np.asfortranarray(w0 ** 2), np.ones(w0.shape)


def rho_of(c):
    return c["rho"] if "rho" in c else c["r"] ** (c["beta"] / c["N"])


def run_oracle_online(name):
    import oracle as O
    c = ONLINE[name]
    fx = load(name)
    v, w0 = make_online_inputs(c)
    check_inputs(fx, v)
    v64 = v.astype(np.float64)
    idx = visit_order(c)
    a0, b0 = initial_stats(c, w0)
    orc = O.Online(w0, beta=c["beta"], r=c["r"], inner_iters=c["iters"], restart=c["restart"], seed=c["seed"],
                   dataset_size=c["N"], dataset=v64 if c["restart"] == "warm" else None)
    kw = dict(a=a0, b=b0, rho=rho_of(c), t=0, commits=0)
    if c["restart"] == "warm":
        kw["warm_h"] = np.full((c["K"], c["N"]), c.get("h0", 1.0))
    orc.set(**kw)
    frames = np.asfortranarray(v64[:, idx.astype(np.int64)])
    tt, to = orc.run(frames, index=idx)
    st = orc.state(warm_h=c["restart"] == "warm")
    return fx, st, tt, to


def run_engine_online(name, record=()):
    """The same case through the device engine, one engine call per recorded
    commit boundary (so the dictionary can be read there)."""
    import paper_1106_4198_b200 as E
    c = ONLINE[name]
    fx = load(name)
    v, w0 = make_online_inputs(c)
    check_inputs(fx, v)
    idx = visit_order(c)
    a0, b0 = initial_stats(c, w0)
    eng = E.Online(c["F"], c["K"], c["beta"], c["iters"], restart=c["restart"], seed=c["seed"],
                   n_store=c["N"] if c["restart"] == "warm" else 0)
    eng.set_dictionary(w0, a0, b0)
    eng.set_counters(0, 0, rho_of(c))
    if c["restart"] == "warm":
        eng.fill_warm_h(c.get("h0", 1.0))
    frames = np.asfortranarray(v[:, idx.astype(np.int64)])
    snaps = {}
    pos = 0
    for rc in sorted(record):
        end = rc * c["beta"]
        eng.run(frames[:, pos:end], index=idx[pos:end])
        snaps[rc] = eng.state()
        pos = end
    eng.run(frames[:, pos:], index=idx[pos:])
    st = eng.state(warm_h=c["restart"] == "warm")
    tr = eng.trace()
    eng.close()
    return fx, st, snaps, tr


def batch_inputs(name):
    c = BATCH[name]
    fx = load(name)
    v, w0, h0 = make_batch_inputs(c)
    check_inputs(fx, v)
    return c, fx, v, w0, h0
