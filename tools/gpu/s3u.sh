#!/usr/bin/env bash
set -u
OUT=gpurun_out/s3u; mkdir -p $OUT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_grid_sort -s 2 -c 1 -o $OUT/grid_msd python tools/prof_sort.py --cfg cfg1 --reps 3 > $OUT/ncu.log 2>&1
echo "ncu $?" >> $OUT/status.txt
