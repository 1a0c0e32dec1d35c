#!/bin/bash
# GPU tests (incl. the 30-pass long run) + the driver's exact bench command.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python3 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_driver.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_driver.log
tail -3 gpurun_out/bench_driver.log
