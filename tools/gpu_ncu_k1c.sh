#!/bin/bash
# ncu --set full (with source) of one K1C launch at config 3, after the same command ran clean
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 1 --frames 409600 --no-e2e --no-cpu --no-compare"
python bench.py $ARGS > gpurun_out/plain_k1c.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:solve_pair -s 120 -c 1 \
    -o gpurun_out/k1c_full python bench.py $ARGS > gpurun_out/ncu_k1c.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_k1c.log
