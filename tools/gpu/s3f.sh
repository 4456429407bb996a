#!/usr/bin/env bash
set -u
OUT=gpurun_out/s3f; mkdir -p $OUT
timeout 300 tools/exp/tune2 30 > $OUT/tune2.jsonl 2>&1; echo "tune2 $?" >> $OUT/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg4 or presorted or all_equal or few_runs" > $OUT/pytest.log 2>&1
echo "pytest $?" >> $OUT/status.txt
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
for L in sorted; do
  timeout 600 ncu $M -k regex:"k_" --log-file $OUT/launches_cfg4_$L.csv python tools/prof_sort.py --cfg cfg4 --layout $L --reps 1 > $OUT/ncu_$L.log 2>&1
  echo "$L $?" >> $OUT/status.txt
done
