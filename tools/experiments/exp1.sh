#!/bin/bash
O=gpurun_out/exp1; mkdir -p $O
for f in 0 1 2 4; do echo "== c2 fill $f"; timeout 300 python tools/quick_perf.py --n 100000 --q 32 --fill $f --reps 3; done > $O/c2_fills.txt 2>&1
for f in 0 2 4; do echo "== c3 fill $f"; timeout 600 python tools/quick_perf.py --n 1000000 --q 64 --fill $f --reps 2; done > $O/c3_fills.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_rows_masked' -s 1 -c 1 -o $O/fill_c2 python tools/quick_perf.py --n 100000 --q 32 --reps 2 > $O/ncu_fill.log 2>&1
