#!/bin/bash
# Full ncu capture of one launch of a kernel without cache flushes between replay passes
# (L2 keeps what the previous kernels / passes left, like in the pipelined run).
K=${1:-fold_commit}; OUT=${2:-prof_k2_warm}
mkdir -p gpurun_out
SMALL="python bench.py --steps 1 --warmup 1 --frames 409600 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --cache-control none --clock-control none --import-source on -k regex:$K -s 20 -c 1 -o gpurun_out/$OUT $SMALL > gpurun_out/ncu_$OUT.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_$OUT.log
