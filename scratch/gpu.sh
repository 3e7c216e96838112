set -u
OUT=gpurun_out/r2c; mkdir -p $OUT
for t in 128 256 384; do timeout 300 python tools/quick_perf.py --n 1000000 --q 64 --reps 3 --bins-threads $t > $OUT/qp_c3_t$t.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_bins -s 1 -c 1 -o $OUT/full_c3_bins python tools/quick_perf.py --n 1000000 --q 64 --reps 2 > $OUT/ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_bins -s 1 -c 1 -o $OUT/full_c2_bins python tools/quick_perf.py --n 100000 --q 32 --reps 2 --fill 7 --bins-threads 128 > $OUT/ncu_c2.log 2>&1
ls $OUT
