#!/bin/bash
# K1C iteration: parity tests, timeline trace, c3 bench (device + e2e)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_k1c.py -x -q > gpurun_out/k1c_tests.log 2>&1; echo "k1c tests rc=$?"; tail -2 gpurun_out/k1c_tests.log
timeout 60 python tools/pc_trace.py 513 50 4096 10 3 > gpurun_out/pc_trace.log 2>&1; echo "trace rc=$?"
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-compare > gpurun_out/ab_k1c.json 2> gpurun_out/ab_k1c.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/ab_k1c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('k1c', round(d['value']/1e6,2), 'M frames/s', 'e2e', round(d['e2e']['value']/1e6,2), 'ms/launch', round(r.get('ms_per_launch',0),4), 'k2_us', round(r.get('k2_us_per_minibatch',0),1))"
