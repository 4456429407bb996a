mkdir -p gpurun_out/r1b
timeout 600 ./build/tune_pass > gpurun_out/r1b/tune.jsonl 2> gpurun_out/r1b/tune.err; echo "tune $?" >> gpurun_out/r1b/status.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r1b/pytest_gpu.log 2>&1; echo "pytest $?" >> gpurun_out/r1b/status.txt
timeout 600 python bench.py --quick --no-cpu > gpurun_out/r1b/bench.json 2> gpurun_out/r1b/bench.err; echo "bench $?" >> gpurun_out/r1b/status.txt
cat gpurun_out/r1b/status.txt
