#!/usr/bin/env bash
set -u
OUT=gpurun_out/s3e; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "few_runs or cfg4 or presorted or all_equal or warp_spec or joint or distinct or equal" > $OUT/pytest.log 2>&1
echo "pytest $?" >> $OUT/status.txt
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
for L in equal sorted reverse; do
  timeout 600 ncu $M -k regex:"k_" --log-file $OUT/launches_cfg4_$L.csv python tools/prof_sort.py --cfg cfg4 --layout $L --reps 1 > $OUT/ncu_$L.log 2>&1
  echo "$L $?" >> $OUT/status.txt
done
timeout 600 ncu $M -k regex:"k_" --log-file $OUT/launches_cfg3.csv python tools/prof_sort.py --cfg cfg3 --reps 1 > $OUT/ncu_cfg3.log 2>&1
echo "cfg3 $?" >> $OUT/status.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench.json 2> $OUT/bench.err
echo "bench $?" >> $OUT/status.txt
