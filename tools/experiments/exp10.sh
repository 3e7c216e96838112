#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "owned or segmented or golden or hashed" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for cfg in "--own 0" "--own 1"; do echo "== c2 $cfg"; timeout 300 python tools/quick_perf.py --n 100000 --q 32 $cfg --reps 3; done > $O/c2.txt 2>&1
for cfg in "--own 0"; do echo "== c3 $cfg"; timeout 600 python tools/quick_perf.py --n 1000000 --q 64 $cfg --reps 2; done > $O/c3.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_owned' -s 1 -c 1 -o $O/own_c2 python tools/quick_perf.py --n 100000 --q 32 --reps 2 > $O/ncu.log 2>&1
timeout 300 nsys --version > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file $O/launches.csv python tools/quick_perf.py --n 100000 --q 32 --reps 2 > $O/ncu_l.log 2>&1
