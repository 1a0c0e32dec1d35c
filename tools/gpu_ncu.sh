#!/bin/bash
# Full ncu capture of one K1 launch (short bench, 1 GPU).
mkdir -p gpurun_out
SMALL="python bench.py --steps 1 --warmup 1 --frames 409600 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 20 -c 1 -o gpurun_out/prof_k1 $SMALL > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_full.log
