mkdir -p gpurun_out/r1h
timeout 600 ./build/tune_pass 1073741824 4 > gpurun_out/r1h/tune.jsonl 2> gpurun_out/r1h/tune.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:onesweep_pass -s 1 -c 1 -o gpurun_out/r1h/aor_full ./build/tune_pass 1073741824 4 > gpurun_out/r1h/ncu.log 2>&1
echo "exit $?"
timeout 600 ./build/tune_pass 1073741824 8 >> gpurun_out/r1h/tune.jsonl 2>> gpurun_out/r1h/tune.err
