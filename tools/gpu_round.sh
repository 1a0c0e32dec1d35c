#!/bin/bash
# One GPU call: GPU tests, then a short bench.  Output under gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 2 --warmup 1 --frames 409600 --no-e2e > gpurun_out/bench_small.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_small.log
tail -5 gpurun_out/bench_small.log
