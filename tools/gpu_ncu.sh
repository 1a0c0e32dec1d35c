#!/bin/bash
# Full ncu capture of one launch of a kernel (short bench, 1 GPU).
# usage: gpu_ncu.sh [kernel-regex] [report-name]
K=${1:-solve_kernel}; OUT=${2:-prof_k1}
mkdir -p gpurun_out
SMALL="python bench.py --steps 1 --warmup 1 --frames 409600 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -s 20 -c 1 -o gpurun_out/$OUT $SMALL > gpurun_out/ncu_$OUT.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_$OUT.log
