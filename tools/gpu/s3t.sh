#!/usr/bin/env bash
set -u
OUT=gpurun_out/s3t; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_small.py -x -q > $OUT/pytest.log 2>&1
echo "pytest $?" >> $OUT/status.txt
timeout 300 python tools/time_small.py > $OUT/time_small.txt 2>&1
echo "time $?" >> $OUT/status.txt
BSORT_GRID_MSD=0 timeout 300 python tools/time_small.py > $OUT/time_small_lsd.txt 2>&1
echo "time0 $?" >> $OUT/status.txt
