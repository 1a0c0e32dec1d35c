"""bench.py's multi-rank plumbing on CPU (gloo, world_size 2): replicas only,
so the only collectives are the barrier and the max over ranks of the timed
region; the reference arm runs on rank 0 alone and the other ranks exit 0."""
import io
import json
import multiprocessing as mp
import os
import socket
import sys
from contextlib import redirect_stdout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, q):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port), BENCH_DIST_BACKEND="gloo")
    sys.path.insert(0, ROOT)
    import bench
    r, w = bench.dist_init()
    bench.barrier(w)
    m = bench.allmax(10.0 * (r + 1) + 0.25, w)
    # the reference arm at a tiny sample: rank 0 prints one JSON line, rank 1 nothing
    args = bench.parse_args(["--impl", "reference", "--config", "c0", "--steps", "1", "--warmup", "1",
                             "--cpu-sample-batches", "1"])
    buf = io.StringIO()
    with redirect_stdout(buf):
        bench.run_reference(args, r, w)
    bench.barrier(w)
    bench.dist_done(w)
    q.put((r, w, m, buf.getvalue()))


def test_two_rank_barrier_allmax_and_reference_arm():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, w0, m0, s0), (r1, w1, m1, s1) = out
    assert (r0, r1, w0, w1) == (0, 1, 2, 2)
    assert m0 == m1 == 20.25
    line = json.loads(s0.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    assert s1 == ""
