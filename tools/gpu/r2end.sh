#!/usr/bin/env bash
# End-of-round-2 evidence: full GPU suite, smoke, bench (+ reference arm), launch list of the
# bench's cfg3 sort (every k_ kernel), small-n timing, ncu --set full of the slowest pass (pass 3,
# k_pass2 half-warp rows) and of the joint histogram sweep.
set -u
OUT=gpurun_out/${1:-r2end}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest $?" >> $OUT/status.txt
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $OUT/smoke.log 2>&1; echo "smoke $?" >> $OUT/status.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench $?" >> $OUT/status.txt
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref $?" >> $OUT/status.txt
timeout 300 python tools/time_small.py 10 14 16 18 20 22 > $OUT/small_n.txt 2>&1; echo "small $?" >> $OUT/status.txt
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
CMD="python bench.py --steps 2 --warmup 3 --quick --no-cpu"
timeout 600 $CMD > $OUT/plain.log 2>&1 && timeout 900 ncu $M -k regex:"k_" --log-file $OUT/launches_bench.csv $CMD > $OUT/ncu_launches.log 2>&1
echo "launches $?" >> $OUT/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pass2 -s 4 -c 1 -o $OUT/pass3_chunked python tools/prof_sort.py --cfg cfg3 --reps 1 > $OUT/ncu_p3.log 2>&1
echo "ncu p3 $?" >> $OUT/status.txt
