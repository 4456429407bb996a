# ncu --set full of the k_pass2 launches of one cfg3 sort (RUN2 pass 2 and stable pass 3)
mkdir -p gpurun_out/p2
timeout 300 python tools/prof_sort.py --cfg cfg3 --reps 1 > gpurun_out/p2/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass2 -s 2 -c 2 -o gpurun_out/p2/prof python tools/prof_sort.py --cfg cfg3 --reps 1 > gpurun_out/p2/ncu.log 2>&1
echo "rc $?"
