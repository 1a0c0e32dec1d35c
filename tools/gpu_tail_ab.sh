#!/bin/bash
# e2e A/B of the chunk-schedule tail divisor (ISNMF_TAIL) at config 3
mkdir -p gpurun_out
for t in 4 8 12; do
ISNMF_TAIL=$t timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-compare > gpurun_out/tail$t.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/tail$t.json').read().strip().splitlines()[-1])
print('tail $t', round(d['value']/1e6,2), 'M frames/s e2e', round(d['e2e']['value']/1e6,3), 'h2d', round(d['e2e']['h2d_gbs'],2))" || tail -5 gpurun_out/tail$t.json
done
