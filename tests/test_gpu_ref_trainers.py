"""The device engine pinned to the REFERENCE's own trainers (tests/golden/
trainer_*.npz, printed by online_resume / batch_train of
/root/reference/proj/include compiled unchanged; see gen_trainer_golden.py)
at the north-star tolerance, 1e-4 relative in fp32: W, A, B at recorded
commits and at the end, the per-commit mini-batch objective trace, pending
statistics of a leftover partial mini-batch, and the stored warm activations.

Cases: config 0 in full; config-0 shape with fresh restarts, r = 0.7
forgetting, CyclingSource order and leftovers; config-1 and config-3
prefixes (config 3 at rho = 0.959670); batch at the config-2 shape (N=2000,
10 epochs, per-epoch objective).
"""
import numpy as np
import pytest

import paper_1106_4198_b200 as E
from trainer_cases import ONLINE, batch_inputs, rel, run_engine_online

pytestmark = pytest.mark.gpu
RTOL = 1e-4


@pytest.mark.parametrize("name", list(ONLINE))
def test_engine_online_matches_reference(name):
    c = ONLINE[name]
    fx, st, snaps, (ts, to, _) = run_engine_online(name, record=c["record"])
    assert st["t"] == int(fx["t"]) and st["commits"] == int(fx["commits"])
    assert st["pending_count"] == int(fx["pending_count"])
    np.testing.assert_array_equal(ts, fx["trace_t"])
    assert rel(to, fx["trace_obj"]) < RTOL, rel(to, fx["trace_obj"])
    for rc, s in snaps.items():
        for k in ("w", "a", "b"):
            assert rel(s[k], fx[f"{k}_{rc}"]) < RTOL, (rc, k, rel(s[k], fx[f"{k}_{rc}"]))
    for k in ("w", "a", "b"):
        assert rel(st[k], fx[k]) < RTOL, (k, rel(st[k], fx[k]))
    if int(fx["pending_count"]):
        for k in ("pending_a", "pending_b"):
            assert rel(st[k], fx[k]) < RTOL, (k, rel(st[k], fx[k]))
        assert rel(st["pending_div"], fx["pending_div"]) < RTOL
    assert rel(st["last_minibatch_obj"], fx["last_minibatch_obj"]) < RTOL
    if "warm_h" in fx:
        keep = fx["warm_h"].shape[1]
        assert rel(st["warm_h"][:, :keep], fx["warm_h"]) < RTOL


def test_engine_batch_matches_reference():
    c, fx, v, w0, h0 = batch_inputs("c2_small")
    out = E.batch_train(v, w0, h0, c["epochs"])
    assert out["epochs"] == int(fx["epochs"])
    assert rel(out["initial_obj"], fx["initial_obj"]) < RTOL
    assert rel(out["obj"], fx["obj"]) < RTOL, rel(out["obj"], fx["obj"])
    assert rel(out["w"], fx["w"]) < RTOL, rel(out["w"], fx["w"])
    assert rel(out["h"][:, :fx["h"].shape[1]], fx["h"]) < RTOL


def test_chunk_stream_source_to_device_matches_reference(tmp_path):
    """ChunkStreamSource -> online_train through the drop-in C++ API on the device
    (tests/cpp/chunk_stream_train.cpp; our ChunkStreamSource feeds the engine
    through its next_block fast path), against the reference's own online_train
    over the same wire stream (irregular chunks, 256-frame permuted buffers)."""
    import subprocess

    from gen_trainer_golden import read_isnm, write_isnm
    from test_cpp_api import build
    from trainer_cases import load, make_online_inputs
    c = ONLINE["c0_chunkstream"]
    fx = load("c0_chunkstream")
    v, w0 = make_online_inputs(c)
    d = tmp_path / "case"
    d.mkdir()
    write_isnm(str(d / "v.isnm"), v.astype(np.float64))
    write_isnm(str(d / "w0.isnm"), w0)
    (d / "params.txt").write_text(f"beta {c['beta']}\niters {c['iters']}\nseed {c['seed']}\n"
                                  f"chunks {c['chunks']}\nbuffer {c['buffer']}\n")
    exe = build("chunk_stream_train", tmp_path)
    r = subprocess.run([exe, str(d)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    st = dict(line.split() for line in open(d / "out_state.txt"))
    assert int(st["t"]) == int(fx["t"]) and int(st["commits"]) == int(fx["commits"])
    tr = np.loadtxt(d / "out_trace.txt", ndmin=2)
    np.testing.assert_array_equal(tr[:, 0].astype(np.uint64), fx["trace_t"])
    assert rel(tr[:, 1], fx["trace_obj"]) < RTOL
    for k in ("w", "a", "b"):
        got = read_isnm(str(d / f"out_{k}.isnm"))
        assert rel(got, fx[k]) < RTOL, (k, rel(got, fx[k]))
    assert rel(float(st["last_minibatch_obj"]), fx["last_minibatch_obj"]) < RTOL
