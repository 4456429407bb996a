mkdir -p gpurun_out/i10
timeout 1200 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/i10/pytest_gpu.log 2>&1; echo "pytest $?"; tail -5 gpurun_out/i10/pytest_gpu.log
timeout 300 python tools/time_small.py 10 13 14 20 > gpurun_out/i10/small.jsonl 2>&1; cat gpurun_out/i10/small.jsonl
