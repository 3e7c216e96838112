#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_validation.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-run > $O/bench.json 2> $O/bench.err
timeout 600 python tools/e2e_threads.py > $O/e2e_thr.txt 2>&1
