#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck, one small sort per kernel family.
set -u
OUT=gpurun_out/${1:-san}; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
env_of() { python -c "import sys; sys.path.insert(0,'tools'); import sanitize_case as s; print(' '.join(f'{k}={v}' for k,v in s.CASES['$1'][2].items()))" 2>/dev/null; }
for tool in memcheck synccheck racecheck; do
  for c in small_cta grid_msd grid_lsd_i64 multilaunch count_u8 count_i16 pass2_ws ws64 joint_chunked; do
    E=$(env_of $c)
    start=$(date +%s)
    env $E BSORT_GRAPH=0 timeout 600 $CS --tool $tool --error-exitcode 9 python tools/sanitize_case.py $c > $OUT/${tool}_$c.log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(( $(date +%s) - start ))s" >> $OUT/status.txt
  done
done
