#!/bin/bash
# K1C quick check: parity suites + c3 bench
O=gpurun_out/k1cq; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_k1c.py tests/test_gpu_trajectory.py tests/test_gpu_ref_trainers.py tests/test_gpu_numerics.py tests/test_gpu_online.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu --no-compare > $O/c3.json 2>&1
python -c "
import json; d=json.loads(open('$O/c3.json').read().strip().splitlines()[-1]); r=d['roofline']
print('c3', round(d['value']/1e6,3), 'M frames/s e2e', round(d['e2e']['value']/1e6,3), 'us/launch', round(r['ms_per_launch']*1e3,1), 'k2', round(r['k2_us_per_minibatch'],1), d['final'])" || tail -5 $O/c3.json
