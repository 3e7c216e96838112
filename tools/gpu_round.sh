#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench lines (ours + reference arm), ncu launch lists
# (c3 headline and c2 secondary), ncu --set full captures of the top kernels.
# Usage (repo root on the box): bash tools/gpu_round.sh TAG [skip-tests]
set -u
TAG=${1:-r2}
SKIP=${2:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
if [ -z "$SKIP" ]; then
  timeout 2400 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
# the sharded (torchrun) path with one rank: peer-memory exchange into its own buffer
PICASSO_FORCE_SHARDED=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 \
   --master-addr 127.0.0.1 --master-port 29555 bench.py --steps 5 --warmup 3 \
   > $OUT/bench_sharded1.json 2> $OUT/bench_sharded1.err
for W in c3 c2; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches_$W.csv \
     python bench.py --workload $W --secondary '' --steps 2 --warmup 3 --no-cpu-baseline --no-clocks --no-run \
     > $OUT/ncu_bench_$W.log 2>&1
done
for spec in c3:k_commute_fr8 c3:k_fill_bins c3:k_owned_fr c2:k_fill_bins c2:k_owned_fr c2:k_commute_fr8; do
  W=${spec%%:*}; k=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
     -o $OUT/full_${W}_$k python bench.py --workload $W --secondary '' --steps 1 --warmup 3 \
     --no-cpu-baseline --no-clocks --no-run > $OUT/ncu_full_${W}_$k.log 2>&1
done
ls -la $OUT
