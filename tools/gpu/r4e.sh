#!/usr/bin/env bash
# A/B of the fixed-trip-count writer loop in k_onesweep_pass_ws (alt_lib/libbsort_wsloop.so) vs the
# plain loop (in-tree): full bench lines (cfg5 local i64 / f64, KV argsort under "configs").
set -u
OUT=gpurun_out/${1:-r4e}; mkdir -p $OUT
for i in 1 2; do
  timeout 900 python bench.py --no-cpu --steps 10 > $OUT/bench_plain_$i.json 2>/dev/null; echo "plain $?" >> $OUT/status.txt
  BSORT_LIB=alt_lib/libbsort_wsloop.so timeout 900 python bench.py --no-cpu --steps 10 > $OUT/bench_wsloop_$i.json 2>/dev/null; echo "wsloop $?" >> $OUT/status.txt
done
# the in-tree build is the expected final state: full GPU suite + smoke on it
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest $? $(tail -1 $OUT/pytest_gpu.log)" >> $OUT/status.txt
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $OUT/smoke.log 2>&1; echo "smoke $?" >> $OUT/status.txt
