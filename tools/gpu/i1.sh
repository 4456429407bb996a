mkdir -p gpurun_out/i1
timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/i1/pytest_gpu.log 2>&1; echo "pytest $?"
tail -3 gpurun_out/i1/pytest_gpu.log
timeout 300 python bench.py --quick --no-cpu > gpurun_out/i1/bench.json 2> gpurun_out/i1/bench.err; echo "bench $?"
cat gpurun_out/i1/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], d['value'], d.get('roofline'))"
BSORT_P2=0 timeout 300 python bench.py --quick --no-cpu > gpurun_out/i1/bench_p2off.json 2>&1; echo "bench0 $?"
cat gpurun_out/i1/bench_p2off.json | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], d['value'])"
timeout 300 python tools/prof_sort.py --cfg cfg3 --reps 1 > gpurun_out/i1/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_(count|onesweep|plan|copy|dist|pass)" --log-file gpurun_out/i1/launches_cfg3.csv python tools/prof_sort.py --cfg cfg3 --reps 1 > /dev/null 2>&1; echo "ncu $?"
