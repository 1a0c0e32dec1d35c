#!/bin/bash
# GPU call: tests (optional), short bench, launch list.  usage: gpu_quick.sh [notest]
mkdir -p gpurun_out
if [ "$1" != "notest" ]; then
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
fi
SMALL="python bench.py --steps 1 --warmup 1 --frames 409600 --no-e2e --no-cpu"
timeout 600 $SMALL > gpurun_out/bench_small.log 2>&1; echo "small rc=$?"; tail -1 gpurun_out/bench_small.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'k1 ms',d['roofline']['ms_per_launch'],'frac',d['roofline']['frac'],'k1share',d['roofline']['k1_share_of_step'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
python tools/launches.py gpurun_out/launches.csv
