mkdir -p gpurun_out/i5
timeout 300 python tools/time_small.py > gpurun_out/i5/small.jsonl 2>&1; echo "t $?"; cat gpurun_out/i5/small.jsonl
BSORT_SMALL=0 timeout 300 python tools/time_small.py > gpurun_out/i5/small0.jsonl 2>&1; echo "t0 $?"; cat gpurun_out/i5/small0.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_small --log-file gpurun_out/i5/ncu_small.csv python tools/time_small.py 16 20 > /dev/null 2>&1; echo "ncu $?"
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/i5/ncu_small.csv")) if len(r)>10]
h=rows[0]; 
import collections
d=collections.defaultdict(list)
for r in rows[1:]:
    x=dict(zip(h,r))
    if x.get("Metric Name")=="gpu__time_duration.sum": d[(x["Kernel Name"][:40], x["Grid Size"])].append(float(x["Metric Value"]))
for k,v in d.items(): print(k, len(v), sorted(v)[len(v)//2])
PY
