#!/usr/bin/env bash
# In-tree build: cfg3 bench (quick) x2, launch list of the pass kernels, parity + small + dist suites.
set -u
OUT=gpurun_out/${1:-r4c}; mkdir -p $OUT
for i in 1 2; do
  timeout 600 python bench.py --quick --no-cpu --steps 10 > $OUT/bench_$i.json 2>/dev/null; echo "bench $?" >> $OUT/status.txt
done
M="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 600 ncu $M -k regex:"k_" --log-file $OUT/launches.csv python tools/prof_sort.py --cfg cfg3 --reps 2 > /dev/null 2>&1; echo "launches $?" >> $OUT/status.txt
timeout 600 ncu $M -k regex:"k_" --log-file $OUT/launches_i64.csv python tools/prof_sort.py --cfg cfg5 --n 1073741824 --reps 1 > $OUT/l64.log 2>&1; echo "launches i64 $?" >> $OUT/status.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_small.py -x -q > $OUT/pytest.log 2>&1; echo "pytest $? $(tail -1 $OUT/pytest.log)" >> $OUT/status.txt
