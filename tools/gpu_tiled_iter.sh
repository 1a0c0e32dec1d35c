#!/bin/bash
# K1M window-tiled statistics planes (staged bulk copies): parity suites + c1/c2/c3-K1M benches
O=gpurun_out/tiled; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_mma.py tests/test_gpu_online.py tests/test_gpu_batch.py tests/test_gpu_kernels.py tests/test_gpu_ref_trainers.py tests/test_gpu_trajectory.py tests/test_gpu_numerics.py tests/test_gpu_heldout.py -x -q > $O/tests.log 2>&1; echo "tests rc=$?"; tail -5 $O/tests.log
timeout 600 python bench.py --config c2 --steps 3 --warmup 1 --no-cpu > $O/bench_c2.log 2>&1; echo "c2 rc=$?"
timeout 300 python bench.py --config c1 --steps 3 --warmup 2 --no-cpu --no-compare > $O/bench_c1.log 2>&1; echo "c1 rc=$?"
ISNMF_K1C=0 timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-compare > $O/bench_c3_k1m.log 2>&1; echo "c3 k1m rc=$?"
for c in c2 c1 c3_k1m; do python - <<PY
import json
d=json.loads(open('$O/bench_$c.log').read().strip().splitlines()[-1]); r=d.get('roofline',{})
print('$c', round(d['value'],1), d['unit'], 'ms/step', round(d['ms_per_step'],2), 'us/launch', round(r.get('ms_per_launch',0)*1e3,1), 'fp32 frac', r.get('fp32_roofline',{}).get('frac'), 'k2', r.get('k2_us_per_minibatch'))
PY
done
