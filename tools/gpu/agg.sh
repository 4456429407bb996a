mkdir -p gpurun_out/agg
timeout 300 python bench.py --quick --no-cpu > gpurun_out/agg/bench.json 2>/dev/null; echo "bench $?"
python -c "import json; d=json.load(open('gpurun_out/agg/bench.json')); print('agg', d['ms_per_step'], d['roofline']['frac'])"
BSORT_P2_AGG=0 timeout 300 python bench.py --quick --no-cpu > gpurun_out/agg/bench0.json 2>/dev/null; echo "bench0 $?"
python -c "import json; d=json.load(open('gpurun_out/agg/bench0.json')); print('noagg', d['ms_per_step'], d['roofline']['frac'])"
timeout 300 python tools/prof_sort.py --cfg cfg3 --reps 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:k_pass2 --log-file gpurun_out/agg/launches.csv python tools/prof_sort.py --cfg cfg3 --reps 1 > /dev/null 2>&1; echo "ncu $?"
python tools/launch_summary.py gpurun_out/agg/launches.csv
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
