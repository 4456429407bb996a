#!/usr/bin/env bash
# launch lists of cfg4 distinct16 / equal and a source-level ncu capture of k_pass2 pass 2 (cfg3)
set -u
OUT=gpurun_out/s3b; mkdir -p $OUT
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
for L in distinct16 equal; do
  timeout 300 python tools/prof_sort.py --cfg cfg4 --layout $L --reps 1 > $OUT/plain_$L.log 2>&1 &&
  timeout 600 ncu $M -k regex:"k_" --log-file $OUT/launches_cfg4_$L.csv python tools/prof_sort.py --cfg cfg4 --layout $L --reps 1 > $OUT/ncu_$L.log 2>&1
  echo "$L $?" >> $OUT/status.txt
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pass2 -s 1 -c 1 -o $OUT/pass2_cfg3 python tools/prof_sort.py --cfg cfg3 --reps 1 > $OUT/ncu_full.log 2>&1
echo "full $?" >> $OUT/status.txt
