#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench lines (ours + reference arm), ncu launch list,
# ncu --set full captures of the top kernels.  Usage (repo root on the box): bash tools/gpu_round.sh TAG
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-clocks --no-run > $OUT/ncu_bench.log 2>&1
for k in k_fill_blk k_owned_fr k_commute_fr2 k_delta; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
     -o $OUT/full_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-clocks --no-run > $OUT/ncu_full_$k.log 2>&1
done
ls -la $OUT
