#!/usr/bin/env bash
# A/B: 32-bit write-out offsets in k_onesweep_pass (alt_lib/libbsort_gofs32.so, -DBSORT_GOFS32) vs in-tree.
set -u
OUT=gpurun_out/${1:-r4a}; mkdir -p $OUT
for i in 1 2; do
  timeout 600 python bench.py --quick --no-cpu --steps 10 > $OUT/bench_base_$i.json 2>/dev/null; echo "base $?" >> $OUT/status.txt
  BSORT_LIB=alt_lib/libbsort_gofs32.so timeout 600 python bench.py --quick --no-cpu --steps 10 > $OUT/bench_gofs32_$i.json 2>/dev/null; echo "gofs32 $?" >> $OUT/status.txt
done
M="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 600 ncu $M -k regex:"k_onesweep_pass" --log-file $OUT/launches_base.csv python tools/prof_sort.py --cfg cfg3 --reps 2 > /dev/null 2>&1; echo "l base $?" >> $OUT/status.txt
BSORT_LIB=alt_lib/libbsort_gofs32.so timeout 600 ncu $M -k regex:"k_onesweep_pass" --log-file $OUT/launches_gofs32.csv python tools/prof_sort.py --cfg cfg3 --reps 2 > /dev/null 2>&1; echo "l gofs32 $?" >> $OUT/status.txt
BSORT_LIB=alt_lib/libbsort_gofs32.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/pytest_parity_gofs32.log 2>&1; echo "pytest parity gofs32 $?" >> $OUT/status.txt
