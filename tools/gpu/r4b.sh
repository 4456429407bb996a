#!/usr/bin/env bash
# Fallback / A-B switches of the LSD path: the parity suite under each of them (the round-1 kernels
# are what runs where bsort_selftest fails, so they must stay bit-exact after the round-2 changes).
set -u
OUT=gpurun_out/${1:-r4b}; mkdir -p $OUT
run() {  # tag, env assignment
  env "$2" timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/parity_$1.log 2>&1
  echo "$1 ($2) rc=$? $(tail -1 $OUT/parity_$1.log)" >> $OUT/status.txt
}
run p2_off BSORT_P2=0
run p2_unchunked BSORT_P2_CHUNKED=0
run ws_off BSORT_WS=0
run no_joint BSORT_NO_JOINT=1
run p2_run2 BSORT_P2_RUN2=1
run graph_off BSORT_GRAPH=0
