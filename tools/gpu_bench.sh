#!/bin/bash
# GPU call: tests, short + full bench, ncu launch list of a short bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
SMALL="python bench.py --steps 1 --warmup 1 --frames 409600 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/bench_small.log 2>&1; echo "small rc=$?"; tail -2 gpurun_out/bench_small.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "full rc=$?"; tail -3 gpurun_out/bench_full.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
