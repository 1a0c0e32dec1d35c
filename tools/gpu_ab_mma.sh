#!/bin/bash
# GPU call: GPU tests, then the short config-3 bench with K1M (default) and with the FFMA kernel (ISNMF_MMA=0).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -15 gpurun_out/pytest_gpu.log
SMALL="python bench.py --steps 2 --warmup 1 --frames 409600 --no-e2e --no-cpu"
for m in 1 0; do
ISNMF_MMA=$m timeout 600 $SMALL > gpurun_out/bench_mma$m.log 2>&1; echo "mma=$m rc=$?"
tail -1 gpurun_out/bench_mma$m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value',d['value'],'k1 ms',r['ms_per_launch'],'frac',r['frac'],'pass',r['pass_frac'],'k2us',r['k2_us_per_minibatch'])"
done
