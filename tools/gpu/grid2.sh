for c in 32 64 96 128 148; do echo "ctas $c"; BSORT_GRID_CTAS=$c timeout 300 python tools/time_small.py 16 18 20 21 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['dtype'], d['n'], d['event_us_single_call'])
"; done
