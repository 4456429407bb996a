mkdir -p gpurun_out/fused
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/fused/pytest.log 2>&1; echo "pytest $?"; tail -5 gpurun_out/fused/pytest.log
timeout 900 python bench.py --force-dist --steps 5 --warmup 3 > gpurun_out/fused/dist1.json 2> gpurun_out/fused/dist1.err; echo "dist $?"; tail -3 gpurun_out/fused/dist1.err
python -c "
import json; d=json.load(open('gpurun_out/fused/dist1.json'))
print(d['ms_per_step'], d['e2e'], d['gpu_launches'])
for k,v in d['configs'].items(): print(k, v)
"
