#!/bin/bash
# Round evidence: smoke, full bench (engine + reference arm), launch list, K1 ncu capture.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_full.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log
SMALL="python bench.py --steps 1 --warmup 1 --frames 409600 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launch.log 2>&1; echo "ncu-list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 20 -c 1 -o gpurun_out/prof_k1 $SMALL > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
