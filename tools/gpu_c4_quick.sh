#!/bin/bash
# c4 quick check: K1T parity suites + c4 bench
O=gpurun_out/c4q; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_online.py tests/test_gpu_heldout.py tests/test_gpu_kernels.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c4" > $O/tests_full.log 2>&1; echo "fullsize rc=$?"; tail -2 $O/tests_full.log
timeout 300 python bench.py --config c4 --steps 4 --warmup 2 --no-cpu --no-compare > $O/c4.json 2>&1
python -c "
import json; d=json.loads(open('$O/c4.json').read().strip().splitlines()[-1]); r=d['roofline']
print('c4', round(d['value']/1e6,3), 'M frames/s e2e', round(d['e2e']['value']/1e6,3), 'us/launch', round(r['ms_per_launch']*1e3,1), 'k2', round(r['k2_us_per_minibatch'],1), d['final'])" || tail -5 $O/c4.json
