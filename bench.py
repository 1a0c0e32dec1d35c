#!/usr/bin/env python3
"""Benchmark of the B200 online IS-NMF engine (BASELINE.json metric).

Metric: online IS-NMF frames/s at F=513, K=50, beta=4096, I=10 (config 3,
"twelve hours" shape: N=2.7M frames, rho=0.99^(beta/1000) per mini-batch,
1 pass = one step) on one B200, plus % of the FP32 roofline.

  value  — frames/s with V resident in HBM (one step = one pass over N frames
           through isnmf_online_run with a device pointer)
  e2e    — the same pass through the same C-ABI call with V in pinned HOST
           memory: the engine streams 64-mini-batch chunks H2D on a copy stream,
           double-buffered; W/A/B and the trace are read back every step
  roofline — K1 (solve_kernel) achieved FP32 TFLOP/s = algorithmic flops per
           launch (6*F*K*(I+1) per frame x frames per launch) / mean launch time
           from CUDA events recorded around every K1 launch on the engine's
           compute stream during the timed region
  cpu_baseline — the CPU fp64 oracle (restatement of the reference; the
           reference itself cannot be compiled: no Eigen) on a bounded prefix.

`--impl reference` times that CPU implementation of the path with all host
threads on a bounded sample per step (rank 0 only under torchrun).
Multi-GPU: replicas only (north_star: one GPU); each rank runs its own pass,
value = sum of frames over ranks / max time over ranks (weak scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from tools.synth import CONFIGS  # noqa: E402

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
# FP32 FMA peak: MEASURED_PEAKS.json carries no FP32 figure, so the denominator is the
# nominal 148 SM x 128 lanes x 2 flop x 1.965 GHz (clocks.max.sm) — the highest the
# part can issue; tools/probe measured 72.4 on this pool (profiles/r01_probe.txt)
FP32_PEAK_NOMINAL = 148 * 128 * 2 * 1.965e9 / 1e12


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="engine", choices=["engine", "reference"])
    p.add_argument("--config", default="c3")
    p.add_argument("--frames", type=int, default=0, help="override N (debug)")
    p.add_argument("--cpu-sample-batches", type=int, default=4)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-compare", action="store_true", help="skip the batch-vs-online comparison")
    return p.parse_args(argv)


parse_args = parse


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": float(self.rows[0][1]),
                "samples": len(self.rows), "reasons": reasons}


_BACKEND = None


def dist_init():
    """One process per GPU (torchrun env).  Replicas only: the collectives are a
    barrier and the max-over-ranks of the timed region, over NCCL on GPU boxes
    (gloo on CPU, or BENCH_DIST_BACKEND)."""
    global _BACKEND
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        _BACKEND = os.environ.get("BENCH_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        if _BACKEND == "nccl":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count())
        dist.init_process_group(_BACKEND)
    return rank, world


def barrier(world):
    if world > 1:
        import torch
        import torch.distributed as dist
        if _BACKEND == "nccl":
            dist.barrier(device_ids=[torch.cuda.current_device()])
        else:
            dist.barrier()


def allmax(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if _BACKEND == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_done(world):
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# useful-product ceiling of 3xTF32 on the legacy mma.sync pipe: m16n8k8 TF32 measured at
# 1020 flop/clk/SM (tools/probe/mma_probe2.cu), 3 MMAs per product, 148 SMs at 1.965 GHz
MMA_3XTF32_PEAK = 1020.0 / 3 * 148 * 1.965e9 / 1e12


def measured_peaks():
    try:
        return json.load(open(MEASURED))
    except (OSError, ValueError):
        return {}


def tcgen05_3xtf32_peak():
    """Useful-product ceiling of 3xTF32 on the 5th-generation tensor cores: the dense tf32
    rate is half the bf16 rate, taken from the MEASURED bf16 burst figure in
    MEASURED_PEAKS.json (else the nominal 2.25 PFLOP/s of B200_PROFILING.md), and every
    useful product costs three tf32 products (hi*hi + hi*lo + lo*hi)."""
    mp = measured_peaks()
    bf16 = mp.get("bf16_tflops")
    src = ("MEASURED_PEAKS.json bf16_tflops %.1f (burst) / 2 (tf32) / 3 (3xTF32)" % bf16 if bf16 else
           "fallback: nominal 2250 TFLOP/s bf16 dense (B200_PROFILING.md) / 2 / 3")
    return (bf16 or 2250.0) / 2.0 / 3.0, src


KERNELS = {
    "K1C": "solve_pair_kernel (K1C: 2-CTA cluster per 56 frames, tcgen05.mma kind::tf32 3xTF32 with TMEM "
           "accumulators and the dictionary rows as TMEM A operand, TMA bulk loads, DSMEM partial exchange)",
    "K1M": "solve_mma_kernel (K1M: 3xTF32 mma.sync for every contraction)",
    "K1": "solve_kernel (FP32 FMA + 3xTF32 mma.sync phase A)",
    "K1T": "solve_large_tc_kernel (K1T: tcgen05 phase B, mma.sync phase A)",
    "K1L": "solve_large_kernel (3xTF32 mma.sync)",
    "generic": "solve_generic_kernel (FP32)",
}


def k1_traffic(config):
    """DRAM bytes per K1 launch of this config from its committed ncu --set full
    capture (profiles/k1_traffic_<config>.json), or None when there is none."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", f"k1_traffic_{config}.json")))
        return d["dram_bytes_read"] + d["dram_bytes_write"], d.get("source")
    except (OSError, ValueError, KeyError):
        return None, None


def cpu_baseline(cfg, v_host_cols, w0, a0, threads, batches):
    """Oracle online pass over a bounded prefix (`batches` mini-batches)."""
    import oracle as O
    F, K, beta, iters = cfg["F"], cfg["K"], cfg["beta"], cfg["iters"]
    n = beta * batches
    sample = np.asfortranarray(v_host_cols[:, :n])
    t0 = time.perf_counter()
    O.baseline_online(sample, w0, a0, a0, beta, iters, cfg["rho"], threads=threads)
    dt = time.perf_counter() - t0
    return n / dt, dt, n


def reference_build_rate(cfg, v_host_cols, w0, a0, frames):
    """The reference's OWN online trainer (online_resume / online_step / dictionary_commit, headers
    compiled unchanged over the test-only Eigen-subset shim: oracle/_ref/ref_trainer, built by
    `make -C oracle ref` where /root/reference exists) on `frames` frames of this shape, 1 core.
    Returns (frames/s, seconds) from the trainer's own loop, or None when the binary is absent."""
    import struct
    import subprocess
    import tempfile
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_trainer")
    if not os.access(exe, os.X_OK):
        return None

    def write_isnm(path, m):
        m = np.asfortranarray(m, dtype=np.float64)
        with open(path, "wb") as f:
            f.write(b"ISNM" + struct.pack("<IQQ", 1, m.shape[0], m.shape[1]))
            f.write(m.tobytes(order="F"))
    try:
        with tempfile.TemporaryDirectory() as d:
            write_isnm(os.path.join(d, "v.isnm"), v_host_cols[:, :frames])
            write_isnm(os.path.join(d, "w0.isnm"), w0)
            with open(os.path.join(d, "params.txt"), "w") as f:
                f.write(f"beta {cfg['beta']}\niters {cfg['iters']}\nrho {cfg['rho']!r}\nrestart warm\nseed 1\n"
                        f"eps 1e-12\nbudget {frames}\na0 {float(a0.flat[0])!r}\nh0 1.0\norder in_order\n")
            subprocess.run([exe, "online", d], check=True, timeout=600, stdout=subprocess.DEVNULL,
                           stderr=subprocess.DEVNULL)
            st = dict(line.split() for line in open(os.path.join(d, "state.txt")))
            sec = float(st["train_seconds"])
            return frames / sec, sec
    except Exception:  # noqa: BLE001 (a reported extra, never fatal to the bench)
        return None


def host_info():
    cpu = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return cpu, os.cpu_count()


def run_reference(args, rank, world):
    cfg = dict(CONFIGS[args.config])
    if rank != 0:
        return
    from tools.synth import spectrogram_np, w_init
    F, K, beta = cfg["F"], cfg["K"], cfg["beta"]
    threads = os.cpu_count() or 1
    batches = max(threads, args.cpu_sample_batches)
    v = spectrogram_np(F, K, beta * batches, seed=1234)
    w0 = w_init(F, K, 4321)
    a0 = np.full((F, K), 1e-3)
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_baseline(cfg, v, w0, a0, threads, 1)
    rates, times = [], []
    for _ in range(args.steps):
        r, dt, n = cpu_baseline(cfg, v, w0, a0, threads, batches)
        rates.append(r)
        times.append(dt)
    val = float(np.mean(rates))
    cpu, ncpu = host_info()
    line = {"impl": "reference", "metric": "online IS-NMF frames/sec (F=513,K=50,beta=4096)", "value": val,
            "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: F={F}, K={K}, beta={beta}, I={cfg['iters']}, "
                                   f"rho={cfg['rho']:.6f}; CPU sample {beta * batches} frames per step",
                       "parallelism": f"{threads} host threads"},
            "cpu_baseline": {"value": val, "unit": "frames/s", "cores": threads, "kind": "port",
                             "sample": f"{batches} mini-batches x {beta} frames of the {args.config} shape "
                                       f"per step; fp64 oracle restatement (reference unbuildable: no Eigen); "
                                       f"{cpu}"},
            "e2e": {"value": val, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_batch_rate(F, K, n_sample, epochs_sample=1):
    """Oracle batch_train (fp64 restatement of batch.hpp:84-143) on a sample of
    n_sample frames: seconds per epoch per frame (the epoch cost is linear in N)."""
    import oracle as O
    from tools.synth import spectrogram_np
    v = spectrogram_np(F, K, n_sample, seed=61).astype(np.float64)
    rng = np.random.default_rng(62)
    w0 = rng.uniform(0.1, 1.0, size=(F, K))
    h0 = rng.uniform(0.1, 1.0, size=(K, n_sample))
    t0 = time.perf_counter()
    O.batch_train(v, w0, h0, epochs_sample)
    dt = time.perf_counter() - t0
    return dt / (epochs_sample * n_sample), dt


def run_batch(args, rank, world):
    """Config 2: batch IS-NMF, 100 MU epochs over F=513 x N=225k (O(FKN) comparison path).
    value = epochs/s from CUDA events around the enqueued epochs (isnmf_batch_profile);
    e2e = the same call with V in pinned host memory, host-timed (V and H uploads, W and
    H downloads included)."""
    import torch

    import paper_1106_4198_b200 as E
    from tools.synth import spectrogram_torch
    dev = int(os.environ.get("LOCAL_RANK", rank)) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev)
    cfg = dict(CONFIGS["c2"])
    F, K, N = cfg["F"], cfg["K"], args.frames or cfg["N"]
    epochs = cfg["epochs"]
    vd = spectrogram_torch(F, K, N, seed=7 + rank, shape=cfg["shape"], device="cuda")
    rng = np.random.default_rng(8 + rank)
    w0 = rng.uniform(0.1, 1.0, size=(F, K))
    h0 = np.asfortranarray(rng.uniform(0.1, 1.0, size=(K, N)))  # column-major, as the C ABI takes it
    torch.cuda.synchronize()
    E.batch_profile(1)
    for _ in range(max(1, args.warmup)):
        E.batch_train(vd, w0, h0, 2)
    times, launches = [], 0
    with ClockSampler(dev) as clk:
        time.sleep(0.5)
        for _ in range(args.steps):
            barrier(world)
            torch.cuda.synchronize()
            out = E.batch_train(vd, w0, h0, epochs)
            ms, nl = E.batch_profile()
            torch.cuda.synchronize()
            barrier(world)
            times.append(allmax(ms, world))
            launches += nl
    t = float(np.sum(times)) / 1e3 / args.steps
    flops = 12.0 * F * K * N * epochs + 2.0 * F * K * N
    peak = FP32_PEAK_NOMINAL
    e2e = None
    if not args.no_e2e:
        vh = torch.empty_like(vd, device="cpu").pin_memory()
        vh.copy_(vd)
        E.batch_train(vh, w0, h0, 1)
        t0 = time.perf_counter()
        calls = []
        for _ in range(args.steps):
            tc = time.perf_counter()
            E.batch_train(vh, w0, h0, epochs)
            calls.append(round(1e3 * (time.perf_counter() - tc), 1))
        e2e_s = allmax((time.perf_counter() - t0) / args.steps, world)
        e2e = {"value": world * epochs / e2e_s, "unit": "epochs/s", "h2d_bytes_per_step": int(N * F * 4 + K * N * 8),
               "d2h_bytes_per_step": int(K * N * 8 + F * K * 8), "calls_ms": calls,
               "timing": "host wall clock of the whole batch_train call with V in pinned host memory"}
    cpu = None
    if rank == 0 and not args.no_cpu:
        n_s = 4000
        spf, dt = cpu_batch_rate(F, K, n_s)
        cpu_name, ncpu = host_info()
        cpu = {"value": 1.0 / (spf * N), "unit": "epochs/s", "cores": 1, "kind": "port",
               "sample": f"1 epoch over {n_s} frames ({dt:.1f} s) of the c2 shape, scaled to N={N} (the epoch "
                         f"cost is linear in N); fp64 oracle restatement of batch.hpp:84-143 on 1 core of "
                         f"{cpu_name} ({ncpu} cores)"}
    if rank == 0:
        print(json.dumps({"metric": "batch IS-NMF epochs/sec (F=513,K=50,N=225k)", "value": world * epochs / t,
                          "unit": "epochs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": 1e3 * t, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                          "dtype": "f32", "data": "synthetic",
                          "config": {"workload": f"c2: F={F}, K={K}, N={N}, {epochs} epochs per step, W0/H0 ~ "
                                                 f"U(0.1,1); V device-resident, device-timed (CUDA events)",
                                     "parallelism": "replicas" if world > 1 else "single",
                                     "l2": "inputs larger than L2 (V = %.2f GB fp32)" % (N * F * 4 / 1e9)},
                          "roofline": {"bound": "tensor", "achieved": flops / t / 1e12, "peak": MMA_3XTF32_PEAK,
                                       "unit": "TFLOP/s", "frac": flops / t / 1e12 / MMA_3XTF32_PEAK,
                                       "kernel": "solve_mma_kernel multi-tile (K1M: 3xTF32 mma.sync) + fold_commit",
                                       "flops_per_step": flops,
                                       "flop_model": "12FKN per epoch (H pass 6FKN + statistics 6FKN; the "
                                                     "objective shares the next epoch's first W h) + 2FKN",
                                       "traffic": k1_traffic("c2")[0], "traffic_source": k1_traffic("c2")[1],
                                       "traffic_unit": "bytes per K1M launch = per epoch (ncu dram__bytes_read+write)",
                                       "algorithmic_bytes_per_launch": float(N) * (4 * F + 8 * K),
                                       "algorithmic_bytes_note": "per epoch: V read once (4F per frame) + H read and "
                                                                 "written in fp32 (8K per frame)",
                                       "peak_source": "mma.sync m16n8k8 tf32 1020 flop/clk/SM (tools/probe/mma_probe2.cu)"
                                                      " / 3 (3xTF32), 148 SM x 1.965 GHz",
                                       "fp32_roofline": {"peak": peak, "frac": flops / t / 1e12 / peak,
                                                         "note": "north_star: FP32 FMA peak, nominal 148 SM x 128 x 2 "
                                                                 "x 1.965 GHz; target >= 50%"}},
                          "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches, "clocks": clk.summary(),
                          "final_obj": float(out["obj"][-1]), "initial_obj": out["initial_obj"]}), flush=True)


def objective_device(vd, w, h, eps=1e-12):
    """(1/N) sum is_term((V - WH) / (eps + WH)) (kernels.hpp:43-55) in fp64 on the device
    (torch; a measurement aid for the comparison below, not the engine)."""
    import torch
    wt = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    ht = torch.from_numpy(np.ascontiguousarray(h)).cuda()
    acc, n = 0.0, vd.shape[0]
    for s0 in range(0, n, 1 << 16):
        x = wt @ ht[:, s0:s0 + (1 << 16)]
        u = (vd[s0:s0 + (1 << 16), :w.shape[0]].T.double() - x) / (eps + x)
        acc += float(torch.clamp(u - torch.log1p(u), min=0.0).sum())
    return acc / n


def batch_vs_online(seed=4040):
    """north_star: batch-vs-online wall-clock on the same data, next to the host CPU.
    Data: the config-2 spectrogram (F=513, N=225k, K*=50) on the device.  Online: K=50,
    config 1's mini-batch beta=1000 and I=10, one pass, rho=1, W0 (l1-normalised
    U(0.1,1)), A0=B0=1e-3, warm H0=1.  Batch: 100 epochs (config 2) from the same W0 and
    H0=1.  Device times from CUDA events; objective = the batch objective of (W, H) with
    H = the online warm store.  CPU: the fp64 oracle on 1 core, projected from samples."""
    import torch

    import paper_1106_4198_b200 as E
    from tools.synth import spectrogram_np, spectrogram_torch, w_init
    F, K, N, beta, iters, epochs = 513, 50, 225_000, 1000, 10, 100
    vd = spectrogram_torch(F, K, N, seed=seed, shape=0.5, device="cuda")
    w0 = w_init(F, K, seed + 1)
    a0 = np.full((F, K), 1e-3)
    eng = E.Online(F, K, beta, iters, restart="warm", n_store=N)
    on_ms = []
    for _ in range(2):  # the first run warms up
        eng.set_dictionary(w0, a0, a0)
        eng.set_counters(0, 0, 1.0)
        eng.fill_warm_h(1.0)
        torch.cuda.synchronize()
        prof = E.Profile(eng, per_kernel=False)
        prof.start()
        eng.enqueue(vd, N, vd.stride(0))
        eng.synchronize()
        on_ms.append(prof.stop()["span_ms"])
    st = eng.state(warm_h=True)
    eng.close()
    on_obj = objective_device(vd, st["w"], st["warm_h"])
    h0 = np.ones((K, N))
    E.batch_profile(1)
    E.batch_train(vd, w0, h0, 2)
    out = E.batch_train(vd, w0, h0, epochs)
    b_ms, _ = E.batch_profile()
    b_obj = np.asarray(out["obj"])
    hit = np.nonzero(b_obj <= on_obj)[0]
    ep_match = int(hit[0]) + 1 if hit.size else None
    del vd
    torch.cuda.empty_cache()
    # CPU (fp64 oracle, 1 core): online frames/s on 4 mini-batches, batch s/epoch/frame on 2000 frames
    import oracle as O
    vs = spectrogram_np(F, K, 4 * beta, seed=seed + 2)
    t0 = time.perf_counter()
    O.baseline_online(vs, w0, a0, a0, beta, iters, 1.0, threads=1)
    cpu_on_fps = 4 * beta / (time.perf_counter() - t0)
    spf, _ = cpu_batch_rate(F, K, 2000)
    cpu_name, _ = host_info()
    return {"data": f"F={F}, N={N}, K*={K} synthetic (config 2's spectrogram)",
            "online": {"config": f"K={K}, beta={beta}, I={iters}, 1 pass, rho=1, warm H0=1, A0=B0=1e-3",
                       "gpu_ms": float(on_ms[-1]), "objective": on_obj,
                       "cpu_1core_s_projected": N / cpu_on_fps},
            "batch": {"config": f"K={K}, {epochs} epochs, H0=1", "gpu_ms": float(b_ms),
                      "objective_after_epochs": float(b_obj[-1]),
                      "epochs_to_reach_online_objective": ep_match,
                      "gpu_ms_to_reach_online_objective": (None if ep_match is None
                                                           else float(b_ms) * ep_match / epochs),
                      "cpu_1core_s_projected": epochs * N * spf},
            "cpu": f"fp64 oracle port, 1 core of {cpu_name}; online timed on {4 * beta} frames, batch on "
                   f"1 epoch of 2000 frames, projected to N={N} (per-frame cost independent of N)"}


def run_engine(args, rank, world):
    import torch

    import paper_1106_4198_b200 as E
    from tools.synth import spectrogram_torch, w_init
    ndev = torch.cuda.device_count()
    dev = int(os.environ.get("LOCAL_RANK", rank)) % max(ndev, 1)
    torch.cuda.set_device(dev)
    cfg = dict(CONFIGS[args.config])
    F, K, beta, iters = cfg["F"], cfg["K"], cfg["beta"], cfg["iters"]
    N = args.frames or cfg["N"]
    rho = cfg["rho"]
    flops_per_frame = 6.0 * F * K * (iters + 1)

    # synthetic V (device) + pinned host copy for e2e
    vd = spectrogram_torch(F, K, N, seed=1000 + rank, shape=cfg["shape"], device="cuda")
    torch.cuda.synchronize()
    w0 = w_init(F, K, 77 + rank)
    a0 = np.full((F, K), 1e-3)

    eng = E.Online(F, K, beta, iters, restart="warm", n_store=N)

    zero_fk = np.zeros((F, K), order="F")

    def reinit():
        """Config 3's initial state (W0, A0 = B0 = 1e-3, no pending statistics, t = commits = 0,
        warm store h0 = 1): every step is exactly one config-3 pass, not a continuation."""
        eng.set_dictionary(w0, a0, a0)
        eng.set_pending(zero_fk, zero_fk, 0.0, 0)  # (the N mod beta leftover frames of the previous pass)
        eng.set_counters(0, 0, rho)
        eng.fill_warm_h(1.0)

    def one_pass(frames):
        eng.enqueue(frames, N, frames.stride(0))

    # warm-up
    for _ in range(args.warmup):
        reinit()
        one_pass(vd)
        eng.synchronize()

    # timed steps: V resident in HBM.  Each step re-initialises the state outside
    # the timed region, then one pass is bracketed by a barrier + device
    # synchronize on both sides and timed with CUDA events on the engine's own
    # compute stream (every engine kernel runs there); value = frames / the sum of
    # the step times (max over ranks).
    launches = 0
    ms_total = 0.0
    wall = 0.0
    with ClockSampler(dev) as clk:
        time.sleep(0.5)  # let nvidia-smi start sampling before the timed region
        for _ in range(args.steps):
            reinit()
            barrier(world)
            torch.cuda.synchronize()
            launches0 = eng.launch_count()
            prof = E.Profile(eng, per_kernel=False)  # events only around the step (per-kernel events cost ~1%)
            prof.start()
            t_wall = time.perf_counter()
            one_pass(vd)
            eng.synchronize()
            kstats = prof.stop()
            torch.cuda.synchronize()
            wall += time.perf_counter() - t_wall
            barrier(world)
            ms_total += allmax(kstats["span_ms"], world)
            launches += eng.launch_count() - launches0
    value = world * N * args.steps / (ms_total / 1e3)
    st = eng.state()

    # roofline of K1: one more pass with events around every launch (not part of `value`)
    reinit()
    kprof = E.Profile(eng, per_kernel=True)
    kprof.start()
    one_pass(vd)
    eng.synchronize()
    kstats = kprof.stop()
    k1_ms = kstats["solve_ms"] / max(1, kstats["solve_launches"])
    frames_per_launch = kstats["solve_frames"] / max(1, kstats["solve_launches"])
    k2_ms = kstats["tail_ms"] / max(1, kstats["solve_launches"])
    achieved = flops_per_frame * frames_per_launch / (k1_ms / 1e3) / 1e12
    peak = FP32_PEAK_NOMINAL

    # e2e: the whole user call through the C ABI with V in pinned HOST memory —
    # initial state pushed (W0/A0/B0 H2D, store fill), the pass (V streamed H2D in
    # chunks on the copy stream, double-buffered), the dictionary read back (D2H)
    e2e = None
    if not args.no_e2e:
        vh = torch.empty_like(vd, device="cpu").pin_memory()
        vh.copy_(vd)
        del vd
        torch.cuda.empty_cache()
        reinit()
        one_pass(vh)
        eng.synchronize()
        wbuf = np.empty((F, K), order="F")
        e2e_s = 0.0
        for _ in range(args.steps):
            barrier(world)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            reinit()
            one_pass(vh)
            eng.synchronize()
            E.lib().isnmf_online_get_dictionary(eng._h, E._p(wbuf), None, None)
            e2e_s += allmax(time.perf_counter() - t0, world)
        e2e = {"value": world * N * args.steps / e2e_s, "unit": "frames/s",
               "h2d_bytes_per_step": int(N * F * 4 + 3 * F * K * 8), "d2h_bytes_per_step": int(F * K * 8),
               "h2d_gbs": N * F * 4 * args.steps / e2e_s / 1e9,
               "timing": "host wall clock per step (state init + pass + W read back), summed over steps"}

    cpu = None
    if rank == 0 and not args.no_cpu:
        from tools.synth import spectrogram_np
        batches = args.cpu_sample_batches
        vs = spectrogram_np(F, K, beta * batches, seed=55)
        r, dt, n = cpu_baseline(cfg, vs, w0, a0, 1, batches)
        cpu_name, ncpu = host_info()
        cpu = {"value": r, "unit": "frames/s", "cores": 1, "kind": "port",
               "sample": f"first {batches} mini-batches ({n} frames, {dt:.1f} s) of the {args.config} shape, "
                         f"fp64 oracle restatement of the reference path on 1 core of {cpu_name} "
                         f"({ncpu} cores); the reference needs Eigen, which is not installed"}
        nref = beta * min(2, batches)
        rb = reference_build_rate(cfg, vs, w0, a0, nref)
        if rb:
            cpu["reference_build"] = {
                "value": rb[0], "unit": "frames/s", "cores": 1, "kind": "reference",
                "sample": f"{nref} frames ({rb[1]:.1f} s in the trainer's own loop): the reference's online_resume "
                          "compiled unchanged over the test-only Eigen-subset shim (oracle/ref), 1 core; the shim "
                          "evaluates eagerly, so real Eigen would be faster - the port above is the stronger baseline"}

    traffic, traffic_src = k1_traffic(args.config)
    compare = None
    if rank == 0 and args.config == "c3" and not args.no_compare:
        compare = batch_vs_online()
    solver = eng.solver()
    if solver in ("K1C", "K1T"):  # tcgen05: the 3xTF32 useful-product ceiling of the tensor cores
        tpeak, tsrc = tcgen05_3xtf32_peak()
    else:  # legacy mma.sync pipe
        tpeak = MMA_3XTF32_PEAK
        tsrc = "mma.sync m16n8k8 tf32 1020 flop/clk/SM (tools/probe/mma_probe2.cu) / 3 (3xTF32), 148 SM x 1.965 GHz"
    pass_tflops = flops_per_frame * N * args.steps / (ms_total / 1e3) / 1e12
    roofline = {"bound": "tensor", "achieved": achieved, "peak": tpeak, "unit": "TFLOP/s", "frac": achieved / tpeak,
                "peak_source": tsrc,
                "kernel": KERNELS.get(solver, solver), "solver": solver,
                "flop_model": "6*F*K*(I+1) useful flops per frame (I MM iterations of Lam = W h, W^T q, W^T r "
                              "plus the statistics pass), fp32-equivalent; the 3xTF32 split products are not counted",
                "flops_per_launch": flops_per_frame * frames_per_launch, "ms_per_launch": k1_ms,
                "traffic": traffic, "traffic_source": traffic_src,
                "traffic_unit": "bytes per launch (ncu dram__bytes_read+write)",
                "algorithmic_bytes_per_launch": frames_per_launch * (4 * F + 16 * K),
                "algorithmic_bytes_note": "per frame: V read once (4F) + the fp64 warm activation read and written (16K)",
                "fp32_roofline": {"peak": peak, "achieved": achieved, "frac": achieved / peak,
                                  "pass_frac": pass_tflops / peak,
                                  "note": "north_star roofline: the pass's flops at the FP32 FMA peak (nominal 148 SM "
                                          "x 128 x 2 x 1.965 GHz = 74.4 TFLOP/s; MEASURED_PEAKS.json has no FP32 "
                                          "entry, tools/probe measured 72.4 on this pool); target >= 50%"},
                "k1_share_of_step": kstats["solve_ms"] / kstats["span_ms"],
                "k2_us_per_minibatch": 1e3 * k2_ms}
    if rank == 0:
        metric = ("online IS-NMF frames/sec (F=513,K=50,beta=4096)" if args.config == "c3" else
                  f"online IS-NMF frames/sec ({args.config}: F={F},K={K},beta={beta})")
        line = {"metric": metric, "value": value, "unit": "frames/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_total / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"{args.config}: F={F}, K={K}, beta={beta}, I={iters}, N={N}, "
                                       f"rho={rho:.6f}; each step = one pass from W0, A0=B0=1e-3, "
                                       f"warm store h0=1 (state re-initialised outside the timed region)",
                           "global_batch": beta, "parallelism": "replicas" if world > 1 else "single",
                           "l2": "inputs larger than L2 (V = %.2f GB fp32)" % (N * F * 4 / 1e9)},
                "roofline": roofline,
                "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches, "batch_vs_online": compare,
                "clocks": clk.summary(), "wall_s": wall,
                "final": {"t": st["t"], "commits": st["commits"], "last_minibatch_obj": st["last_minibatch_obj"]}}
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world = dist_init()
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.config == "c2":
        run_batch(args, rank, world)
    else:
        run_engine(args, rank, world)
    dist_done(world)


if __name__ == "__main__":
    main()
