#!/bin/bash
# Box probe run on the GPU host: device, FP32 FMA peak, PCIe, host CPU.
mkdir -p gpurun_out
{
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
nproc; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node"
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
SMI=$!
./tools/probe/probe
kill $SMI
} > gpurun_out/probe.log 2>&1
cat gpurun_out/probe.log
