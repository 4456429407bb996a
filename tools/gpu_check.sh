#!/usr/bin/env bash
# One gpurun call: GPU parity tests (+ optional full-size), per-kernel launch lists for cfg3 and
# cfg4/distinct16, the bench, and the pass tuner.  Usage: bash tools/gpu_check.sh TAG [full]
mkdir -p gpurun_out/$1
timeout 1500 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/$1/pytest_gpu.log 2>&1; echo "pytest $?"
if [ "$2" = "full" ]; then
  timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/$1/pytest_full.log 2>&1; echo "pytest full $?"
fi
for spec in "--cfg cfg3" "--cfg cfg4 --layout distinct16"; do
  tag=$(echo $spec | tr -d ' -')
  timeout 300 python tools/prof_sort.py $spec --reps 1 > gpurun_out/$1/plain_$tag.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_(count|onesweep|plan|copy|dist)" \
     --log-file gpurun_out/$1/launches_$tag.csv python tools/prof_sort.py $spec --reps 1 > /dev/null 2>&1
  echo "$tag $?"
done
timeout 900 python bench.py --no-cpu > gpurun_out/$1/bench.json 2> gpurun_out/$1/bench.err; echo "bench $?"
timeout 300 ./build/tune_pass 1073741824 4 > gpurun_out/$1/tune.jsonl 2> gpurun_out/$1/tune.err; echo "tune $?"
