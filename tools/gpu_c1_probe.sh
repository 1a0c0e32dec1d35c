mkdir -p gpurun_out
timeout 120 python tools/mm_timeline.py 513 20 1000 10 > gpurun_out/mm_c1.log 2>&1; echo "tl rc=$?"
for nw in 12 8; do ISNMF_MMA_WARPS=$nw timeout 300 python bench.py --config c1 --steps 3 --warmup 2 --no-e2e --no-cpu --no-compare > gpurun_out/c1_nw$nw.json 2>&1; echo "nw $nw rc=$?"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"solve|fold" -c 400 --csv --log-file gpurun_out/launches_c1.csv python bench.py --config c1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-compare > /dev/null 2>&1; echo "ncu rc=$?"
