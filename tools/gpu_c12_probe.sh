#!/bin/bash
# c1 / c2 timelines (lib_prof) and K1 time vs inner iterations at the c1 shape
O=gpurun_out/c12; mkdir -p $O
timeout 200 python tools/mm_timeline.py 513 20 1000 10 > $O/mm_c1.log 2>&1; echo "c1 tl rc=$?"
timeout 200 python tools/batch_timeline.py 3 > $O/batch_tl.log 2>&1; echo "c2 tl rc=$?"
timeout 300 python tools/k1_time.py 513 20 1000 1 513 20 1000 5 513 20 1000 10 > $O/k1_time_c1.log 2>&1; echo "k1_time rc=$?"
cat $O/k1_time_c1.log
