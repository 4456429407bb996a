mkdir -p gpurun_out/i4
timeout 900 python -m pytest tests/test_gpu_small.py -x -q > gpurun_out/i4/pytest_small.log 2>&1; echo "small $?"; tail -15 gpurun_out/i4/pytest_small.log
timeout 300 python tools/sweep_n.py 24 1 > gpurun_out/i4/sweep_small.jsonl 2>&1; echo "sweep $?"
BSORT_SMALL=0 timeout 300 python tools/sweep_n.py 24 1 > gpurun_out/i4/sweep_nosmall.jsonl 2>&1; echo "sweep0 $?"
python - <<'PY'
import json
a=[json.loads(l) for l in open("gpurun_out/i4/sweep_small.jsonl") if l.startswith("{")]
b=[json.loads(l) for l in open("gpurun_out/i4/sweep_nosmall.jsonl") if l.startswith("{")]
for x,y in zip(a,b): print(x["cfg"], x["dtype"], x["n"], round(x["median_ms"]*1000,1), "us  vs", round(y["median_ms"]*1000,1))
PY
