#!/bin/bash
# round-2 bench lines for every config + the reference arm (profiles/r04_bench_*.json)
mkdir -p gpurun_out
for c in c1 c4; do
  extra=""; [ $c = c4 ] && extra="--cpu-sample-batches 1"
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 $extra > gpurun_out/r04_bench_$c.log 2>&1
  echo "$c rc=$?"; tail -1 gpurun_out/r04_bench_$c.log | cut -c1-200
done
timeout 600 python bench.py --config c2 --steps 3 --warmup 1 > gpurun_out/r04_bench_c2.log 2>&1; echo "c2 rc=$?"
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r04_bench_c3.log 2>&1; echo "c3 rc=$?"
tail -1 gpurun_out/r04_bench_c3.log | cut -c1-300
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r04_bench_reference.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/r04_bench_reference.log | cut -c1-300
