#!/bin/bash
# K1C vs K1M at config 3 (device-timed bench, no CPU/e2e legs), then the -m gpu suite
mkdir -p gpurun_out
ARGS="--steps 5 --warmup 3 --no-e2e --no-cpu --no-compare"
timeout 300 python bench.py $ARGS > gpurun_out/ab_k1c.json 2> gpurun_out/ab_k1c.err; echo "k1c rc=$?"
ISNMF_K1C=0 timeout 300 python bench.py $ARGS > gpurun_out/ab_k1m.json 2> gpurun_out/ab_k1m.err; echo "k1m rc=$?"
for f in ab_k1c ab_k1m; do python -c "
import json,sys; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', round(d['value']/1e6,2), 'M frames/s', 'ms/launch', round(r.get('ms_per_launch',0),4), 'k2_us', round(r.get('k2_us_per_minibatch',0),1), 'share', round(r.get('k1_share_of_step',0),3))"; done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_k1c.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_k1c.log
