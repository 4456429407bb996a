#!/usr/bin/env bash
# One gpurun call: build check, GPU parity tests, smoke, bench, ncu launch list + one full
# capture of the dominant kernel.  Usage (from the repo root, under gpurun):
#   bash tools/gpu_round.sh [tag] [what...]     what in {tests, smoke, bench, launches, full}
set -u
TAG=${1:-r1}
shift || true
WHAT=${*:-"tests smoke bench launches full"}
mkdir -p gpurun_out
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$OUT/gpu.txt" 2>&1
has() { case " $WHAT " in *" $1 "*) return 0;; esac; return 1; }

if has tests; then
  timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest gpu exit $?" >> "$OUT/status.txt"
fi
if has smoke; then
  timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > "$OUT/smoke.log" 2>&1
  echo "smoke exit $?" >> "$OUT/status.txt"
fi
if has bench; then
  timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
  echo "bench exit $?" >> "$OUT/status.txt"
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
  echo "bench ref exit $?" >> "$OUT/status.txt"
fi
CMD="python bench.py --steps 2 --warmup 3 --quick --no-cpu"
if has launches; then
  timeout 600 $CMD > "$OUT/plain.log" 2>&1 &&
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv -k regex:"k_" \
      --log-file "$OUT/launches.csv" $CMD > "$OUT/ncu_launches.log" 2>&1
  echo "ncu launches exit $?" >> "$OUT/status.txt"
fi
if has full; then
  PCMD="python tools/prof_sort.py --cfg cfg3 --reps 1"
  timeout 600 $PCMD > "$OUT/plain_prof.log" 2>&1 &&
  # launch 4 of one cfg3 sort = pass 3, the stable (slowest) pass, k_onesweep_pass_ws (0: pass 0,
  # 1-2: the two pass-1 variants, 3: pass 2)
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:onesweep_pass -s 4 -c 1 \
      -o "$OUT/pass" $PCMD > "$OUT/ncu_full.log" 2>&1
  echo "ncu full pass exit $?" >> "$OUT/status.txt"
fi
cat "$OUT/status.txt"
