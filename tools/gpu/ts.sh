timeout 600 python tools/time_small.py 10 12 13 14 15 16 17 18 20 22
BSORT_SMALL_MAX=20480 timeout 300 python tools/time_small.py 14
BSORT_GRAPH=0 timeout 300 python tools/time_small.py 16 20
