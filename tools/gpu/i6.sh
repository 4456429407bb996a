mkdir -p gpurun_out/i6
timeout 900 python -m pytest tests/test_gpu_small.py -x -q > gpurun_out/i6/pytest_small.log 2>&1; echo "small $?"; tail -5 gpurun_out/i6/pytest_small.log
timeout 300 python tools/time_small.py 16 18 20 21 22 > gpurun_out/i6/small.jsonl 2>&1; echo "t $?"; cat gpurun_out/i6/small.jsonl
for c in 1024 4096; do BSORT_SMALL_CHUNK=$c timeout 300 python tools/time_small.py 16 18 20 > gpurun_out/i6/small_c$c.jsonl 2>&1; echo "chunk $c"; cat gpurun_out/i6/small_c$c.jsonl; done
