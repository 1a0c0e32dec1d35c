#!/bin/bash
# c4 iteration: K1T statistics chain (ISNMF_CHAIN CTAs per plane) parity + bench A/B
O=gpurun_out/c4; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_online.py tests/test_gpu_heldout.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c4" > $O/tests_full.log 2>&1; echo "fullsize rc=$?"; tail -3 $O/tests_full.log
for g in ${CHAINS:-8 16 0}; do
ISNMF_CHAIN=$g timeout 300 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu --no-compare > $O/c4_chain$g.json 2>&1
python -c "
import json; d=json.loads(open('$O/c4_chain$g.json').read().strip().splitlines()[-1]); r=d['roofline']
print('chain $g', r.get('solver'), round(d['value']/1e6,3), 'M frames/s e2e', round(d['e2e']['value']/1e6,3), 'us/launch', round(r['ms_per_launch']*1e3,1), 'k2', round(r['k2_us_per_minibatch'],1))" || tail -5 $O/c4_chain$g.json
done
