#!/bin/bash
# Round-2 (session 6, after the K1C h^T / frame-ownership, K2 and prefetch changes) evidence: -m gpu suite, smoke, driver c3 bench, reference arm, other configs,
# launch list and ncu --set full of the c3 solve kernel (K1C).  Output under gpurun_out/r13/.
O=gpurun_out/r13; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_c3.log 2>&1; echo "c3 rc=$?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_reference.log 2>&1; echo "ref rc=$?"
ISNMF_K1C=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-compare > $O/bench_c3_k1m.log 2>&1; echo "c3 k1m rc=$?"
for c in c1 c4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 > $O/bench_$c.log 2>&1; echo "$c rc=$?"; done
timeout 600 python bench.py --config c2 --steps 3 --warmup 1 > $O/bench_c2.log 2>&1; echo "c2 rc=$?"
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu --no-compare"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"solve|fold|fresh|fill" -c 1500 --csv \
    --log-file $O/launches_c3.csv python bench.py $ARGS > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:solve_pair -s 700 -c 1 \
    -o $O/k1c_c3_full python bench.py $ARGS > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
