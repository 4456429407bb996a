mkdir -p gpurun_out/r1i
timeout 1500 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/r1i/pytest_gpu.log 2>&1; echo "pytest $?"
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q --durations=20 > gpurun_out/r1i/pytest_full.log 2>&1; echo "pytest full $?"
timeout 900 python bench.py --no-cpu > gpurun_out/r1i/bench.json 2> gpurun_out/r1i/bench.err; echo "bench $?"
