set -x
tag=${1:-v4}
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5 > gpurun_out/pytest_$tag.log
for b in 32 128 256; do timeout 120 python tools/bench_scan.py --beams $b >> gpurun_out/scan_$tag.jsonl 2>>gpurun_out/scan_$tag.err; done
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 5 > gpurun_out/step_$tag.json 2>>gpurun_out/step_$tag.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:env_step_kernel -s 3 -c 1 -o gpurun_out/prof_step_$tag python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ncu_step_$tag.log 2>&1
cat gpurun_out/pytest_$tag.log
