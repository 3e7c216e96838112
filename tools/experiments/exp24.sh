#!/bin/bash
# block fill: parity + geometry sweep at c2, c3
TAG=${TAG:-exp24}; mkdir -p gpurun_out/$TAG
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "block or fill_variants" > gpurun_out/$TAG/pytest.log 2>&1
tail -3 gpurun_out/$TAG/pytest.log
python tools/quick_perf.py --reps 3 --fill 0 2>&1 | grep "rep 2" | sed 's/^/seg default: /'
for tg in ${C2GEOM:-256x4 128x8 64x16 512x2}; do
  set -- ${tg/x/ }
  timeout 120 python tools/quick_perf.py --reps 3 --fill 5 --blk-threads $1 --blk-groups $2 --check 2>&1 | grep "rep 2\|check" | tr '\n' ' ' | sed "s/^/blk $1x$2: /"; echo
done
python tools/quick_perf.py --n 1000000 --q 64 --reps 2 --fill 0 2>&1 | grep "rep 1" | sed 's/^/c3 seg: /'
for tg in ${C3GEOM:-512x16 1024x8 128x16 256x8}; do
  set -- ${tg/x/ }
  timeout 300 python tools/quick_perf.py --n 1000000 --q 64 --reps 2 --fill 5 --blk-threads $1 --blk-groups $2 2>&1 | grep "rep 1" | sed "s/^/c3 blk $1x$2: /"
done
