#!/bin/bash
# K2 change check: broad parity suites + c3 / c1 / c4 benches
O=gpurun_out/k2ab; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_debug_build.py -k "not fullsize and not longrun" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
for c in c3 c1 c4; do
timeout 300 python bench.py --config $c --steps 6 --warmup 3 --no-cpu --no-compare > $O/$c.json 2>&1
python -c "
import json; d=json.loads(open('$O/$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$c', round(d['value']/1e6,3), 'M frames/s e2e', round(d['e2e']['value']/1e6,3), 'us/launch', round(r['ms_per_launch']*1e3,1), 'k2', round(r['k2_us_per_minibatch'],1))" || tail -5 $O/$c.json
done
