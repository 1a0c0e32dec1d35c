#!/bin/bash
# SM clock / power while the online path runs (is a variant power- or clock-limited?)
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 100 > gpurun_out/clk.csv &
SMI=$!
sleep 1
python tools/debug_timing.py 2457600 | tail -2
kill $SMI
sort gpurun_out/clk.csv | uniq -c | sort -rn | head -8
