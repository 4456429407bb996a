timeout 1200 python -m pytest tests/test_gpu_small.py -x -q 2>&1 | tail -3
timeout 600 python tools/time_small.py 13 14 15 16 17 18 19 20 21 22
BSORT_GRID_CHUNK=2048 timeout 300 python tools/time_small.py 16 20
BSORT_GRID_CHUNK=8192 timeout 300 python tools/time_small.py 16 20
