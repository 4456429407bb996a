# round-2 evidence: bench (headline, no profiler), launch list of one cfg3 sort, ncu --set full of
# the slowest pass (k_pass2 pass 3) and of the unstable pass 0; counting-path launch lists
mkdir -p gpurun_out/r2
timeout 600 python bench.py --no-cpu --steps 20 --warmup 3 > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err; echo "bench $?"
head -c 400 gpurun_out/r2/bench.json; echo
timeout 300 python tools/prof_sort.py --cfg cfg3 --reps 1 > gpurun_out/r2/plain.log 2>&1; echo "plain $?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2/launches_cfg3.csv python tools/prof_sort.py --cfg cfg3 --reps 1 > /dev/null 2>&1; echo "launches $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass2 -s 3 -c 1 -o gpurun_out/r2/pass3_full python tools/prof_sort.py --cfg cfg3 --reps 1 > gpurun_out/r2/ncu_full.log 2>&1; echo "full $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_onesweep_pass -c 1 -o gpurun_out/r2/pass0_full python tools/prof_sort.py --cfg cfg3 --reps 1 > gpurun_out/r2/ncu_full0.log 2>&1; echo "full0 $?"
for dt in uint8 int16; do
  timeout 300 python tools/prof_sort.py --cfg cfg2 --dtype $dt --reps 1 > /dev/null 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none --csv --log-file gpurun_out/r2/launches_cfg2_$dt.csv python tools/prof_sort.py --cfg cfg2 --dtype $dt --reps 1 > /dev/null 2>&1; echo "cfg2 $dt $?"
done
