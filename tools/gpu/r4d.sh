#!/usr/bin/env bash
# After the look-back-region fix: the whole parity suite under the round-1 fallback switches.
set -u
OUT=gpurun_out/${1:-r4d}; mkdir -p $OUT
run() {  # tag, env assignments...
  local tag=$1; shift
  env "$@" timeout 900 python -m pytest tests/test_gpu_parity.py -q > $OUT/parity_$tag.log 2>&1
  echo "$tag ($*) rc=$? $(tail -1 $OUT/parity_$tag.log)" >> $OUT/status.txt
}
run p2_off BSORT_P2=0
run p2_ws_off BSORT_P2=0 BSORT_WS=0
run p2_off_unchunked_nojoint BSORT_P2=0 BSORT_NO_JOINT=1
