#!/usr/bin/env bash
# Full-tile split restricted to 32-bit keys-only sorts: one full bench line, then the GPU suite.
set -u
OUT=gpurun_out/${1:-r4f}; mkdir -p $OUT
timeout 600 python bench.py --no-cpu --steps 10 > $OUT/bench.json 2>/dev/null; echo "bench $?" >> $OUT/status.txt
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest $? $(tail -1 $OUT/pytest_gpu.log)" >> $OUT/status.txt
timeout 200 python -c 'import __graft_entry__ as g; g.smoke()' > $OUT/smoke.log 2>&1; echo "smoke $?" >> $OUT/status.txt
