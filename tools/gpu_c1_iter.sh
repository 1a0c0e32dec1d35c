#!/bin/bash
# c1 iteration: K1M/K1P parity suites, c1 bench (device + e2e) with K1P on and off
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mma.py tests/test_gpu_online.py tests/test_gpu_ref_trainers.py tests/test_gpu_trajectory.py -x -q > gpurun_out/c1_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c1_tests.log
for p in 1 0; do
ISNMF_K1P=$p timeout 300 python bench.py --config c1 --steps 3 --warmup 2 --no-cpu --no-compare > gpurun_out/c1_k1p$p.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/c1_k1p$p.json').read().strip().splitlines()[-1]); r=d['roofline']
print('k1p $p', r.get('solver'), round(d['value']/1e6,2), 'M frames/s e2e', round(d['e2e']['value']/1e6,2), 'ms/launch', round(r['ms_per_launch']*1e3,1), 'k2', round(r['k2_us_per_minibatch'],1))" || tail -5 gpurun_out/c1_k1p$p.json
done
