set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5 > gpurun_out/pytest_v3.log
for rm in 8 16 24 32; do SPARROW_REFILL_MIN=$rm timeout 120 python tools/bench_scan.py >> gpurun_out/scan_v3.jsonl 2>>gpurun_out/scan_v3.err; done
for rm in 16 24; do SPARROW_REFILL_MIN=$rm timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/step_v3_$rm.json 2>>gpurun_out/step_v3.err; done
timeout 120 python tools/bench_scan.py --reps 3 > gpurun_out/plain_scan.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:env_scan_kernel -s 4 -c 1 -o gpurun_out/prof_scan_v3 python tools/bench_scan.py --reps 3 > gpurun_out/ncu_scan_v3.log 2>&1
cat gpurun_out/pytest_v3.log
