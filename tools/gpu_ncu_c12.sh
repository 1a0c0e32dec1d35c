#!/bin/bash
# ncu --set full of one K1P launch at config 1 and one batch K1M (multi-tile) launch at config 2
O=gpurun_out/c12ncu; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:solve_mma -s 300 -c 1 \
    -o $O/k1p_c1_full python bench.py --config c1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-compare > $O/ncu_c1.log 2>&1; echo "ncu c1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:solve_mma -s 2 -c 1 \
    -o $O/k1m_c2_full python tools/batch_once.py 4 > $O/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"solve|fold" -c 600 --csv \
    --log-file $O/launches_c1.csv python bench.py --config c1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-compare > /dev/null 2>&1; echo "launch list c1 rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"solve|fold" -c 60 --csv \
    --log-file $O/launches_c2.csv python tools/batch_once.py 20 > /dev/null 2>&1; echo "launch list c2 rc=$?"
