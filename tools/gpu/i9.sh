timeout 900 python -m pytest tests/test_gpu_small.py -x -q 2>&1 | tail -30
timeout 300 python tools/time_small.py 10 12 13 14 20
