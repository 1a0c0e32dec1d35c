#!/bin/bash
# Configs 1 and 2 with K1M (ISNMF_MMA=1) and with the FFMA kernels (ISNMF_MMA=0).
mkdir -p gpurun_out
for m in 1 0; do
for c in c1; do ISNMF_MMA=$m timeout 900 python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_${c}_m$m.log 2>&1; echo "$c mma=$m rc=$?"; tail -1 gpurun_out/bench_${c}_m$m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('value',d['value'],'k1 ms',r.get('ms_per_launch'),'frac',r['frac'],'k2us',r.get('k2_us_per_minibatch'))"; done
ISNMF_MMA=$m timeout 900 python bench.py --config c2 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c2_m$m.log 2>&1; echo "c2 mma=$m rc=$?"; tail -1 gpurun_out/bench_c2_m$m.log | cut -c1-300
done
