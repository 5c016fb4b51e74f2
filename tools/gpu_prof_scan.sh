tag=${1:-ps}
timeout 120 python tools/bench_scan.py --reps 3 > gpurun_out/plain_scan_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:env_scan_kernel -s 4 -c 1 -o gpurun_out/prof_scan_$tag python tools/bench_scan.py --reps 3 > gpurun_out/ncu_scan_$tag.log 2>&1
echo rc=$?
