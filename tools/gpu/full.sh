mkdir -p gpurun_out/full
timeout 900 python bench.py > gpurun_out/full/bench.json 2> gpurun_out/full/bench.err; echo "bench $?"
python -c "
import json; d=json.load(open('gpurun_out/full/bench.json'))
print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'] if d['cpu_baseline'] else None, d['clocks'])
for k,v in d.get('configs',{}).items(): print(k, {a: (round(b,4) if isinstance(b,float) else b) for a,b in v.items()})
"
timeout 300 python tools/prof_sort.py --cfg cfg4 --layout equal --reps 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none --csv -k regex:"k_(onesweep|plan|copy)" --log-file gpurun_out/full/launches_cfg4_equal.csv python tools/prof_sort.py --cfg cfg4 --layout equal --reps 1 > /dev/null 2>&1; echo "ncu $?"
python tools/launch_summary.py gpurun_out/full/launches_cfg4_equal.csv
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none --csv -k regex:"k_(onesweep|plan|copy)" --log-file gpurun_out/full/launches_cfg4_reverse.csv python tools/prof_sort.py --cfg cfg4 --layout reverse --reps 1 > /dev/null 2>&1; echo "ncu $?"
python tools/launch_summary.py gpurun_out/full/launches_cfg4_reverse.csv
