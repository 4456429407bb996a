#!/usr/bin/env bash
# sort_host_to tests, full bench (pipelined e2e), k_pass2 visibility under an ncu filter.
set -u
OUT=gpurun_out/${1:-r3c}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "host" > $OUT/pytest_host.log 2>&1; echo "pytest host $?" >> $OUT/status.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench $?" >> $OUT/status.txt
timeout 300 python tools/prof_sort.py --cfg cfg3 --reps 1 > $OUT/plain_prof.log 2>&1; echo "plain prof $?" >> $OUT/status.txt
timeout 600 ncu -k regex:k_nothing -c 1 python tools/prof_sort.py --cfg cfg3 --reps 1 > $OUT/ncu_nothing.log 2>&1; echo "ncu nothing $?" >> $OUT/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pass2 -s 5 -c 1 -o $OUT/pass3_chunked python tools/prof_sort.py --cfg cfg3 --reps 1 > $OUT/ncu_p3.log 2>&1
echo "ncu p3 $?" >> $OUT/status.txt
