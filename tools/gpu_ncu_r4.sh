#!/bin/bash
# round-2 profiles of the config-3 bench: plain run, launch list (engine kernels), one
# ncu --set full capture of K1M; then the full -m gpu suite
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu --no-compare"
python bench.py $ARGS > gpurun_out/plain_c3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"solve|fold|fresh|fill" -c 1500 --csv \
    --log-file gpurun_out/launches_c3.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
python bench.py $ARGS > gpurun_out/plain_c3b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:solve_mma -s 700 -c 1 \
    -o gpurun_out/k1m_c3_r4 python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_all.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_all.log
tail -5 gpurun_out/pytest_gpu_all.log
