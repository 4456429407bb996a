mkdir -p gpurun_out/fso
free -g; nproc; grep -m1 "model name" /proc/cpuinfo
SECONDS=0; timeout 1500 python -m pytest tests/test_gpu_fullsize_oracle.py -x -q --durations=10 > gpurun_out/fso/pytest.log 2>&1; echo "rc $? after $SECONDS s"
tail -16 gpurun_out/fso/pytest.log
