#!/usr/bin/env bash
# Skew-variant (half-warp rows) k_pass2 shapes A/B: in-tree 640x15 vs alt builds; ncu capture of pass 3.
set -u
OUT=gpurun_out/${1:-r3d}; mkdir -p $OUT
for i in 1 2; do
  timeout 600 python bench.py --quick --no-cpu --steps 10 > $OUT/bench_s640x15_$i.json 2>/dev/null; echo "s640x15 $?" >> $OUT/status.txt
  for tag in s512x19 s512x21 s768x13; do
    BSORT_LIB=alt_lib/libbsort_$tag.so timeout 600 python bench.py --quick --no-cpu --steps 10 > $OUT/bench_${tag}_$i.json 2>/dev/null; echo "$tag $?" >> $OUT/status.txt
  done
done
M="--metrics gpu__time_duration.sum --clock-control none --csv"
for tag in s512x19 s512x21 s768x13; do
  BSORT_LIB=alt_lib/libbsort_$tag.so timeout 600 ncu $M -k regex:"k_pass2" --log-file $OUT/launches_$tag.csv python tools/prof_sort.py --cfg cfg3 --reps 2 > /dev/null 2>&1; echo "launches $tag $?" >> $OUT/status.txt
done
timeout 600 ncu $M -k regex:"k_pass2" --log-file $OUT/launches_s640x15.csv python tools/prof_sort.py --cfg cfg3 --reps 2 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pass2 -s 4 -c 1 -o $OUT/pass3_chunked python tools/prof_sort.py --cfg cfg3 --reps 1 > $OUT/ncu_p3.log 2>&1
echo "ncu p3 $?" >> $OUT/status.txt
