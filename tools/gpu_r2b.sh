#!/bin/bash
# batch rework check: batch/online GPU tests, c2 bench, default bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_ref_trainers.py tests/test_gpu_kernels.py tests/test_gpu_heldout.py tests/test_gpu_online.py -q -x > gpurun_out/pytest_b.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_b.log
tail -5 gpurun_out/pytest_b.log
timeout 600 python bench.py --config c2 --steps 3 --warmup 1 > gpurun_out/bench_c2.log 2>&1
echo "bench c2 rc=$?" >> gpurun_out/bench_c2.log
tail -3 gpurun_out/bench_c2.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3.log 2>&1
echo "bench c3 rc=$?" >> gpurun_out/bench_c3.log
tail -3 gpurun_out/bench_c3.log
