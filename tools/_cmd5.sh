mkdir -p gpurun_out/r1g
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r1g/pytest_gpu.log 2>&1; echo "pytest $?"
timeout 900 python bench.py --no-cpu > gpurun_out/r1g/bench.json 2> gpurun_out/r1g/bench.err; echo "bench $?"
