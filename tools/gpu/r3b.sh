#!/usr/bin/env bash
# Software-pipelined joint-histogram sweep A/B (HIST_PIPE=1 in-tree vs alt_lib/libbsort_nopipe.so).
set -u
OUT=gpurun_out/${1:-r3b}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
for i in 1 2; do
timeout 600 python bench.py --quick --no-cpu --steps 10 > $OUT/bench_pipe_$i.json 2> $OUT/bench_pipe_$i.err; echo "bench pipe $?" >> $OUT/status.txt
BSORT_LIB=alt_lib/libbsort_nopipe.so timeout 600 python bench.py --quick --no-cpu --steps 10 > $OUT/bench_nopipe_$i.json 2> $OUT/bench_nopipe_$i.err; echo "bench nopipe $?" >> $OUT/status.txt
done
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 600 ncu $M -k regex:"k_" --log-file $OUT/launches_pipe.csv python tools/prof_sort.py --cfg cfg3 --reps 2 > $OUT/ncu_l.log 2>&1; echo "launches $?" >> $OUT/status.txt
BSORT_LIB=alt_lib/libbsort_nopipe.so timeout 600 ncu $M -k regex:"k_onesweep_hist" --log-file $OUT/launches_nopipe.csv python tools/prof_sort.py --cfg cfg3 --reps 2 > $OUT/ncu_l2.log 2>&1; echo "launches nopipe $?" >> $OUT/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/pytest_parity.log 2>&1; echo "pytest parity $?" >> $OUT/status.txt
