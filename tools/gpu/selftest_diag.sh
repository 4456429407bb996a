#!/usr/bin/env bash
# Is the lane-order self-test stable?  Plain, and inside an ncu session that does not profile it.
set -u
OUT=gpurun_out/${1:-stdiag}; mkdir -p $OUT
./tools/exp/selftest_probe 10 > $OUT/probe_plain.txt 2>&1
timeout 300 ncu -k regex:k_nothing -c 1 ./tools/exp/selftest_probe 5 > $OUT/probe_ncu_unprofiled.txt 2>&1
timeout 300 ncu -k regex:k_probe -c 1 ./tools/exp/selftest_probe 3 > $OUT/probe_ncu_profiled.txt 2>&1
python -c 'import paper_2603_08929_b200 as B; print("selftest", B.selftest())' > $OUT/py_plain.txt 2>&1
timeout 300 ncu -k regex:k_nothing -c 1 python -c 'import paper_2603_08929_b200 as B; print("selftest", B.selftest())' > $OUT/py_ncu.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pass2 -s 5 -c 1 -o $OUT/pass3_chunked python tools/prof_sort.py --cfg cfg3 --reps 1 > $OUT/ncu_p3.log 2>&1
echo "ncu p3 $?" >> $OUT/status.txt
