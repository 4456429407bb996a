mkdir -p gpurun_out/i3
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "strong_p2 or cfg5_local" > gpurun_out/i3/pytest.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/i3/pytest.log
timeout 900 python bench.py --force-dist --steps 5 --warmup 3 > gpurun_out/i3/dist1.json 2> gpurun_out/i3/dist1.err; echo "dist $?"; tail -5 gpurun_out/i3/dist1.err; head -c 3000 gpurun_out/i3/dist1.json
