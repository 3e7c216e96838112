#!/bin/bash
for cfg in ${CFGS:-"192 0" "192 1" "192 2" "256 2" "128 3" "160 2" "192 3"}; do
  set -- ${cfg/_/ }
  timeout 300 python tools/quick_perf.py --n 1000000 --q 64 --reps 3 --fill 7 --bins-threads $1 --bins-shift $2 2>&1 | grep "rep 2" | sed "s/^/c3 bins $1 shift$2: /"
done
