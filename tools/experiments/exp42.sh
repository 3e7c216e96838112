#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bins or fill_variants" 2>&1 | tail -2
for t in 128 256 512; do timeout 120 python tools/quick_perf.py --reps 3 --fill 7 --bins-threads $t 2>&1 | grep "rep 2" | sed "s/^/c2 bins $t: /"; done
timeout 300 python tools/quick_perf.py --n 1000000 --q 64 --reps 2 --fill 6 2>&1 | grep "rep 1" | sed "s/^/c3 seg: /"
for t in 128 256 512; do timeout 300 python tools/quick_perf.py --n 1000000 --q 64 --reps 2 --fill 7 --bins-threads $t 2>&1 | grep "rep 1" | sed "s/^/c3 bins $t: /"; done
timeout 300 python tools/quick_perf.py --n 1000000 --q 64 --reps 1 --fill 7 --check 2>&1 | grep "check"
