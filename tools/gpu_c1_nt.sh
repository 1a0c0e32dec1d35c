#!/bin/bash
# c1 A/B: frames per K1M CTA (ISNMF_MMA_NT)
mkdir -p gpurun_out
for nt in 1 10 14 16 20; do
ISNMF_MMA_NT=$nt timeout 300 python bench.py --config c1 --steps 3 --warmup 2 --no-e2e --no-cpu --no-compare > gpurun_out/c1_nt$nt.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/c1_nt$nt.json').read().strip().splitlines()[-1]); r=d['roofline']
print('nt $nt', round(d['value']/1e6,2), 'M frames/s ms/launch', round(r['ms_per_launch']*1e3,1), 'k2', round(r['k2_us_per_minibatch'],1))"
done
