#!/bin/bash
# Round-end style GPU call: tests, smoke, full c3 bench + reference arm, other
# configs, launch list of a short bench, ncu --set full of K1.  Output under gpurun_out/.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
for c in c1 c2 c4; do timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; done
SMALL="python bench.py --steps 1 --warmup 1 --frames 409600 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
python tools/launches.py gpurun_out/launches.csv
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${K1:-solve_mma_kernel} -s 20 -c 1 -o gpurun_out/prof_k1_full $SMALL > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
