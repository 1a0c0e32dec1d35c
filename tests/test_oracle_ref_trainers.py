"""The fp64 oracle's trainers pinned to the REFERENCE's own trainers.

tests/golden/trainer_*.npz hold trajectories printed by the reference's
online_resume / dictionary_commit / online_step (online.hpp:254-419) and
batch_train (batch.hpp:84-143), compiled unchanged from
/root/reference/proj/include over the Eigen-subset shim (gen_trainer_golden.py).
Both sides compute in fp64 and differ only in summation order inside the
products, so the bound is 1e-12 relative after up to 100 commits / 10 epochs
(measured: ~4e-15 on W, A, B and the trace; ||dW||_F, a difference of nearby
dictionaries, ~2e-14).

Cases: config 0 in full (warm restarts from H0 = 1, A0 = B0 = 1e-3); the
config-0 shape with fresh restarts (seeded mt19937_64 init), forgetting
r = 0.7, the reference's CyclingSource order and a leftover partial
mini-batch after 2.5 passes; config-1 and config-3 prefixes (5 and 4
mini-batches, config 3 with rho = 0.99^(4096/1000)); the batch path at the
config-2 shape with N = 2000 for 10 epochs.
"""
import numpy as np
import pytest

import oracle as O
from trainer_cases import BATCH, ONLINE, batch_inputs, rel, run_oracle_online

TOL = 1e-12


@pytest.mark.parametrize("name", list(ONLINE))
def test_oracle_online_matches_reference(name):
    fx, st, tt, to = run_oracle_online(name)
    c = ONLINE[name]
    assert st["t"] == int(fx["t"]) and st["commits"] == int(fx["commits"])
    assert st["pending_count"] == int(fx["pending_count"])
    np.testing.assert_array_equal(tt, fx["trace_t"])
    assert rel(to, fx["trace_obj"]) < TOL
    for k in ("w", "a", "b"):
        assert rel(st[k], fx[k]) < TOL, (k, rel(st[k], fx[k]))
    if int(fx["pending_count"]):
        for k in ("pending_a", "pending_b"):
            assert rel(st[k], fx[k]) < TOL, k
        assert rel(st["pending_div"], fx["pending_div"]) < TOL
    else:
        assert not np.any(st["pending_a"]) and not np.any(fx["pending_a"])
    assert rel(st["last_minibatch_obj"], fx["last_minibatch_obj"]) < TOL
    assert rel(st["last_delta"], fx["last_delta"]) < 1e-10  # a difference of nearby W's
    assert rel(st["rho"], fx["rho"]) < 1e-15
    if "warm_h" in fx:
        keep = fx["warm_h"].shape[1]
        assert rel(st["warm_h"][:, :keep], fx["warm_h"]) < TOL
    assert c["budget"] == int(fx["t"])


def test_oracle_batch_matches_reference():
    c, fx, v, w0, h0 = batch_inputs("c2_small")
    out = O.batch_train(v.astype(np.float64), w0, h0, c["epochs"])
    assert out["epochs"] == int(fx["epochs"]) == c["epochs"]
    assert rel(out["initial_obj"], fx["initial_obj"]) < TOL
    assert rel(out["obj"], fx["obj"]) < TOL
    assert rel(out["w"], fx["w"]) < TOL
    assert rel(out["h"][:, :fx["h"].shape[1]], fx["h"]) < TOL


def test_fixtures_cover_the_baseline_shapes():
    assert {(c["F"], c["K"], c["beta"], c["iters"]) for c in ONLINE.values()} >= {
        (257, 10, 100, 5), (513, 20, 1000, 10), (513, 50, 4096, 10)}
    assert (BATCH["c2_small"]["F"], BATCH["c2_small"]["K"]) == (513, 50)
