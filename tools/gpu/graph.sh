timeout 900 python -m pytest tests/test_gpu_small.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 300 python tools/time_small.py 10 14 16 18 20 22 24
BSORT_GRAPH=0 timeout 300 python tools/time_small.py 20
./tools/exp/launch_cost 1048576
