#!/bin/bash
# round-2 re-entry check at HEAD: driver bench command, smoke, the -m gpu suite
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r5_bench_c3.log 2>&1; echo "c3 rc=$?"
tail -1 gpurun_out/r5_bench_c3.log | cut -c1-400
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r5_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r5_pytest_gpu.log
