#!/usr/bin/env bash
set -u
OUT=gpurun_out/s3q; mkdir -p $OUT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pass2 -s 1 -c 1 -o $OUT/pass2_chunked python tools/prof_sort.py --cfg cfg3 --reps 1 > $OUT/ncu_p2.log 2>&1
echo "ncu p2 $?" >> $OUT/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pass2 -s 5 -c 1 -o $OUT/pass3_chunked python tools/prof_sort.py --cfg cfg3 --reps 1 > $OUT/ncu_p3.log 2>&1
echo "ncu p3 $?" >> $OUT/status.txt
