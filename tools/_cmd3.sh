mkdir -p gpurun_out/r1c
timeout 600 ./build/tune_pass 1073741824 4 > gpurun_out/r1c/tune.jsonl 2> gpurun_out/r1c/tune.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:onesweep_pass -s 7 -c 1 -o gpurun_out/r1c/ballot ./build/tune_pass 1073741824 4 > gpurun_out/r1c/ncu.log 2>&1
echo "exit $?"
timeout 600 ./build/tune_pass 1073741824 8 >> gpurun_out/r1c/tune.jsonl 2>> gpurun_out/r1c/tune.err
