#!/bin/bash
O=gpurun_out/exp8; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "segmented or owned_fill or golden or hashed" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for cfg in "--fill 0" "--fill 0 --seg-warps 2" "--fill 0 --seg-bits 53248" "--fill 0 --seg-bits 28672" "--fill 3"; do echo "== c2 $cfg"; timeout 300 python tools/quick_perf.py --n 100000 --q 32 $cfg --reps 3; done > $O/c2.txt 2>&1
for cfg in "--fill 0" "--fill 0 --seg-bits 61440" "--fill 0 --seg-bits 126976 --seg-warps 2"; do echo "== c3 $cfg"; timeout 600 python tools/quick_perf.py --n 1000000 --q 64 $cfg --reps 2; done > $O/c3.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_fill_seg' -s 1 -c 1 -o $O/seg_c2 python tools/quick_perf.py --n 100000 --q 32 --reps 2 > $O/ncu.log 2>&1
