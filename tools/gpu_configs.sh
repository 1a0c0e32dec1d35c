#!/bin/bash
mkdir -p gpurun_out
for c in c1 c4; do timeout 900 python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/bench_$c.log | cut -c1-400; done
timeout 900 python bench.py --config c2 --steps 1 > gpurun_out/bench_c2.log 2>&1; echo "c2 rc=$?"; tail -1 gpurun_out/bench_c2.log
