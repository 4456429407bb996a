#!/usr/bin/env bash
set -u
OUT=gpurun_out/s3i; mkdir -p $OUT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_onesweep_hist_joint -c 1 -o $OUT/hist_cfg3 python tools/prof_sort.py --cfg cfg3 --reps 1 > $OUT/ncu_hist.log 2>&1
echo "hist $?" >> $OUT/status.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_count_hist16 -c 1 -o $OUT/hist16 python tools/prof_sort.py --cfg cfg2 --dtype int16 --reps 1 > $OUT/ncu_h16.log 2>&1
echo "h16 $?" >> $OUT/status.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_count_hist8 -c 1 -o $OUT/hist8 python tools/prof_sort.py --cfg cfg2 --dtype uint8 --reps 1 > $OUT/ncu_h8.log 2>&1
echo "h8 $?" >> $OUT/status.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench.json 2> $OUT/bench.err
echo "bench $?" >> $OUT/status.txt
