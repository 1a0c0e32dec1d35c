#!/bin/bash
# ncu --set full of one K1P launch at config 1 (mid-run), summary under gpurun_out/c1ncu/
O=gpurun_out/c1ncu; mkdir -p $O
ARGS="--config c1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-compare"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:solve_mma -s 300 -c 1 \
    -o $O/k1p_c1_full python bench.py $ARGS > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py $O/k1p_c1_full.ncu-rep 40 > $O/k1p_c1_summary.txt 2>&1; tail -60 $O/k1p_c1_summary.txt
