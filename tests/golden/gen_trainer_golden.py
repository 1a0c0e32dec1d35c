"""Regenerates tests/golden/trainer_*.npz: trajectories of the REFERENCE's own
trainers (online_resume / dictionary_commit / online_step, online.hpp:254-419;
batch_train, batch.hpp:84-143), run here by oracle/_ref/ref_trainer =
oracle/ref/ref_trainer.cpp compiled against /root/reference/proj/include
unchanged plus the Eigen-subset shim oracle/ref/eigen_shim (Eigen is absent
from this image).  This container only: /root/reference is not on the GPU box,
so the outputs are committed as fixtures.

Inputs are the BASELINE.json synthetic spectrograms (tools/synth.py,
spectrogram_np / w_init with the seeds below); each fixture stores the
sha256 of its V so a test detects a generator change instead of failing
parity.  usage: python tests/golden/gen_trainer_golden.py
"""
import hashlib
import os
import struct
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from tools.synth import spectrogram_np, w_init  # noqa: E402

BIN = os.path.join(ROOT, "oracle", "_ref", "ref_trainer")

# name: online cases.  a0 = A0 = B0 fill, h0 = warm store fill (BASELINE.json's
# initial state); record = commits whose W/A/B are stored; keep = warm_h columns stored
ONLINE = {
    # config 0 (the CPU-runnable case), one full pass, warm restarts from H0 = 1
    "c0_warm": dict(F=257, K=10, N=10_000, beta=100, iters=5, r=1.0, restart="warm", seed=1, vseed=101,
                    wseed=102, a0=1e-3, h0=1.0, order="in_order", budget=10_000, record=[1, 10, 50], keep=1000),
    # config-0 shape, fresh restarts (the seeded mt19937_64 init, online.hpp:294-301), forgetting
    # rho = r^(beta/N) with r = 0.7, CyclingSource order (online.hpp:53-94), 2.5 passes with a
    # leftover partial mini-batch, reference-default A0 = delta W0^2, B0 = delta
    "c0_fresh_cycling": dict(F=257, K=10, N=1_050, beta=100, iters=5, r=0.7, restart="fresh", seed=7, vseed=103,
                             wseed=104, order="cycling", budget=2_625, record=[5, 20], keep=0),
    # config-0 shape streamed through the reference's ChunkStreamSource (online.hpp:151-220):
    # the wire format [u64 count | count x F f64] in irregular chunks, buffered and permuted
    # per 256-frame buffer; a stream has no size (rho = 1) and no dataset (fresh restarts)
    "c0_chunkstream": dict(F=257, K=10, N=3_000, beta=100, iters=5, r=1.0, restart="fresh", seed=11, vseed=111,
                           wseed=112, order="chunkstream", chunks="37,100,250,3", buffer=256, budget=3_000,
                           record=[7], keep=0),
    # config 1 prefix (F=513, K=20, beta=1000, I=10): first 5 mini-batches
    "c1_prefix": dict(F=513, K=20, N=5_000, beta=1000, iters=10, r=1.0, restart="warm", seed=1, vseed=105,
                      wseed=106, a0=1e-3, h0=1.0, order="in_order", budget=5_000, record=[1, 3], keep=1000),
    # config 3 prefix (F=513, K=50, beta=4096, I=10, rho = 0.99^(4096/1000)): first 4 mini-batches
    "c3_prefix": dict(F=513, K=50, N=16_384, beta=4096, iters=10, r=1.0, rho=0.99 ** (4096 / 1000),
                      restart="warm", seed=1, vseed=107, wseed=108, a0=1e-3, h0=1.0, order="in_order",
                      budget=16_384, record=[1], keep=512),
}
# batch (config-2 shape at reduced N): F=513, K=50, W0, H0 ~ U(0.1, 1)
BATCH = {
    "c2_small": dict(F=513, K=50, N=2_000, epochs=10, vseed=109, wseed=110, keep=500),
}


def write_isnm(path, m):
    m = np.asfortranarray(m, dtype=np.float64)
    with open(path, "wb") as f:
        f.write(b"ISNM" + struct.pack("<IQQ", 1, m.shape[0], m.shape[1]))
        f.write(m.tobytes(order="F"))


def read_isnm(path):
    with open(path, "rb") as f:
        head = f.read(24)
        assert head[:4] == b"ISNM"
        _, r, c = struct.unpack("<IQQ", head[4:])
        return np.frombuffer(f.read(), dtype="<f8").reshape((r, c), order="F").copy()


def vhash(v32):
    return hashlib.sha256(np.asfortranarray(v32, dtype=np.float32).tobytes(order="F")).hexdigest()


def make_online_inputs(c):
    v = spectrogram_np(c["F"], c["K"], c["N"], seed=c["vseed"])
    w0 = w_init(c["F"], c["K"], c["wseed"])
    return v, w0


def make_batch_inputs(c):
    v = spectrogram_np(c["F"], c["K"], c["N"], seed=c["vseed"])
    rng = np.random.default_rng(c["wseed"])
    w0 = np.asfortranarray(rng.uniform(0.1, 1.0, size=(c["F"], c["K"])))
    h0 = np.asfortranarray(rng.uniform(0.1, 1.0, size=(c["K"], c["N"])))
    return v, w0, h0


def run_online(name, c):
    v, w0 = make_online_inputs(c)
    with tempfile.TemporaryDirectory() as d:
        write_isnm(os.path.join(d, "v.isnm"), v.astype(np.float64))
        write_isnm(os.path.join(d, "w0.isnm"), w0)
        keys = ["beta", "iters", "r", "rho", "restart", "seed", "budget", "a0", "h0", "order", "chunks", "buffer"]
        with open(os.path.join(d, "params.txt"), "w") as f:
            for k in keys:
                if k in c:
                    f.write(f"{k} {c[k]!r}\n".replace("'", ""))
            f.write("eta 0\n")
            f.write("record " + ",".join(str(x) for x in c["record"]) + "\n")
        subprocess.run([BIN, "online", d], check=True)
        tr = np.loadtxt(os.path.join(d, "trace.txt"), ndmin=2)
        st = dict(line.split() for line in open(os.path.join(d, "state.txt")))
        out = dict(trace_t=tr[:, 0].astype(np.uint64), trace_obj=tr[:, 1], trace_delta=tr[:, 2],
                   v_sha256=np.array(vhash(v)), params=np.array(repr(c)))
        for k in ("w", "a", "b", "pending_a", "pending_b"):
            out[k] = read_isnm(os.path.join(d, f"{k}.isnm"))
        for rc in c["record"]:
            for k in ("w", "a", "b"):
                out[f"{k}_{rc}"] = read_isnm(os.path.join(d, f"{k}_{rc}.isnm"))
        if c["restart"] == "warm" and c["keep"]:
            out["warm_h"] = read_isnm(os.path.join(d, "warm_h.isnm"))[:, :c["keep"]]
        for k in ("t", "commits", "pending_count"):
            out[k] = np.uint64(int(st[k]))
        for k in ("last_minibatch_obj", "last_delta", "pending_div", "rho"):
            out[k] = np.float64(float(st[k]))
    np.savez_compressed(os.path.join(HERE, f"trainer_{name}.npz"), **out)
    print(name, "commits", int(out["commits"]), "obj", float(out["last_minibatch_obj"]))


def run_batch(name, c):
    v, w0, h0 = make_batch_inputs(c)
    with tempfile.TemporaryDirectory() as d:
        write_isnm(os.path.join(d, "v.isnm"), v.astype(np.float64))
        write_isnm(os.path.join(d, "w0.isnm"), w0)
        write_isnm(os.path.join(d, "h0.isnm"), h0)
        with open(os.path.join(d, "params.txt"), "w") as f:
            f.write(f"epochs {c['epochs']}\neta 0\n")
        subprocess.run([BIN, "batch", d], check=True)
        tr = np.loadtxt(os.path.join(d, "trace.txt"), ndmin=2)
        st = dict(line.split() for line in open(os.path.join(d, "state.txt")))
        out = dict(obj=tr[:, 1], delta=tr[:, 2], w=read_isnm(os.path.join(d, "w.isnm")),
                   h=read_isnm(os.path.join(d, "h.isnm"))[:, :c["keep"]], v_sha256=np.array(vhash(v)),
                   params=np.array(repr(c)), initial_obj=np.float64(float(st["initial_obj"])),
                   epochs=np.uint64(int(st["epoch"])))
    np.savez_compressed(os.path.join(HERE, f"trainer_{name}.npz"), **out)
    print(name, "epochs", int(out["epochs"]), "obj", out["obj"][-1])


if __name__ == "__main__":
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    only = sys.argv[1:]
    for name, c in ONLINE.items():
        if not only or name in only:
            run_online(name, c)
    for name, c in BATCH.items():
        if not only or name in only:
            run_batch(name, c)
