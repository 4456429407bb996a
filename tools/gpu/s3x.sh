#!/usr/bin/env bash
set -u
OUT=gpurun_out/s3x; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > $OUT/pytest.log 2>&1
echo "pytest $?" >> $OUT/status.txt
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 600 ncu $M -k regex:"k_" --log-file $OUT/launches_cfg3.csv python tools/prof_sort.py --cfg cfg3 --reps 1 > $OUT/ncu_cfg3.log 2>&1
echo "cfg3 $?" >> $OUT/status.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --quick > $OUT/bench.json 2> $OUT/bench.err
echo "bench $?" >> $OUT/status.txt
