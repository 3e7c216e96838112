#!/bin/bash
# block fill: list capacity / CTA size sweep at c2
for cfg in "128 8 0" "128 8 2400" "128 8 3072" "128 8 -1" "96 16 0" "96 16 2400" "160 8 0" "64 16 2048"; do
  set -- $cfg
  timeout 120 python tools/quick_perf.py --reps 4 --fill 5 --blk-threads $1 --blk-groups $2 --blk-ecap $3 2>&1 | grep "rep 3" | sed "s/^/blk $1x$2 ecap $3: /"
done
