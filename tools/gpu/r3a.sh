#!/usr/bin/env bash
# Chunked RUN2 pass 2 A/B (BSORT_P2_RUN2=1 vs default) + cooperative-groups grid barrier (cfg1).
set -u
OUT=gpurun_out/${1:-r3a}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
BSORT_P2_RUN2=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_small.py -x -q > $OUT/pytest_run2.log 2>&1; echo "pytest run2 $?" >> $OUT/status.txt
BSORT_P2_RUN2=1 timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cfg3_full or cfg4_full" > $OUT/pytest_full_run2.log 2>&1; echo "pytest full run2 $?" >> $OUT/status.txt
timeout 300 python tools/time_small.py 16 18 20 > $OUT/small.txt 2>&1; echo "small $?" >> $OUT/status.txt
BSORT_GRID_CG=0 timeout 300 python tools/time_small.py 20 > $OUT/small_cg0.txt 2>&1; echo "small cg0 $?" >> $OUT/status.txt
for i in 1 2; do
timeout 600 python bench.py --quick --no-cpu --steps 10 > $OUT/bench_default_$i.json 2> $OUT/bench_default_$i.err; echo "bench default $?" >> $OUT/status.txt
BSORT_P2_RUN2=1 timeout 600 python bench.py --quick --no-cpu --steps 10 > $OUT/bench_run2_$i.json 2> $OUT/bench_run2_$i.err; echo "bench run2 $?" >> $OUT/status.txt
done
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
BSORT_P2_RUN2=1 timeout 600 ncu $M -k regex:"k_" --log-file $OUT/launches_run2.csv python tools/prof_sort.py --cfg cfg3 --reps 2 > $OUT/ncu_l.log 2>&1; echo "launches $?" >> $OUT/status.txt
BSORT_P2_RUN2=1 timeout 600 ncu $M -k regex:"k_" --log-file $OUT/launches_run2_d16.csv python tools/prof_sort.py --cfg cfg4 --layout distinct16 --reps 2 > $OUT/ncu_l2.log 2>&1; echo "launches d16 $?" >> $OUT/status.txt
