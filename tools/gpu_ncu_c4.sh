#!/bin/bash
# Full ncu capture of one K1L launch at config 4.
mkdir -p gpurun_out
SMALL="python bench.py --config c4 --steps 1 --warmup 1 --frames 81920 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/plain_c4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:solve_large -s 5 -c 1 -o gpurun_out/prof_k1l $SMALL > gpurun_out/ncu_k1l.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_k1l.log
