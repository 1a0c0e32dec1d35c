#!/bin/bash
# ncu --set full of one K1T launch (and the K2 after it) at config 4 + launch list
O=gpurun_out/c4; mkdir -p $O
SMALL="python bench.py --config c4 --steps 1 --warmup 1 --frames 81920 --no-e2e --no-cpu --no-compare"
timeout 600 $SMALL > $O/plain_c4.log 2>&1 || { echo plain failed; tail -5 $O/plain_c4.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"solve|fold" -c 200 --csv \
    --log-file $O/launches_c4.csv $SMALL > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"solve_large|fold_commit" -s 10 -c 2 -o $O/k1t_c4_full $SMALL > $O/ncu_k1t.log 2>&1
echo "rc=$?"; tail -2 $O/ncu_k1t.log
