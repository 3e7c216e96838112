#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
for i in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline --no-run > $O/bench_clk_$i.json 2>&1; done
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-run --no-clocks > $O/bench_noclk_$i.json 2>&1; done
timeout 300 python tools/quick_perf.py --n 100000 --q 32 --reps 5 > $O/qp.txt 2>&1
