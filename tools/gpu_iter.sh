#!/bin/bash
# Quick GPU iteration: online/kernel parity tests, then the short config-3 bench for each ISNMF_MMA_WARPS given.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_online.py tests/test_gpu_kernels.py tests/test_gpu_batch.py -m gpu -q -x > gpurun_out/pytest_iter.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_iter.log
SMALL="python bench.py --steps 2 --warmup 1 --frames 409600 --no-e2e --no-cpu"
for w in ${@:-12}; do
ISNMF_MMA_WARPS=$w timeout 600 $SMALL > gpurun_out/bench_iter$w.log 2>&1; echo "warps=$w bench rc=$?"
tail -1 gpurun_out/bench_iter$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value',d['value'],'k1 ms',r['ms_per_launch'],'frac',r['frac'],'pass',r['pass_frac'],'k2us',r['k2_us_per_minibatch'])"
done
