#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for cfg in "--own-direct 1" "--own-direct 0"; do echo "== c2 $cfg"; timeout 300 python tools/quick_perf.py --n 100000 --q 32 $cfg --reps 3; done > $O/c2.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_owned' -s 1 -c 1 -o $O/own_c2 python tools/quick_perf.py --n 100000 --q 32 --reps 2 > $O/ncu.log 2>&1
