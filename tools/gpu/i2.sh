mkdir -p gpurun_out/i2
timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/i2/pytest_gpu.log 2>&1; echo "pytest $?"
tail -5 gpurun_out/i2/pytest_gpu.log
timeout 300 python tools/time_tophist.py > gpurun_out/i2/tophist.log 2>&1; echo "tophist $?"; cat gpurun_out/i2/tophist.log
timeout 300 python bench.py --quick --no-cpu > gpurun_out/i2/bench.json 2> gpurun_out/i2/bench.err; echo "bench $?"
head -c 600 gpurun_out/i2/bench.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dist_tophist -c 1 -o gpurun_out/i2/tophist python tools/time_tophist.py > gpurun_out/i2/ncu_tophist.log 2>&1; echo "ncu $?"
