# Full measurement pass (round-end style): bench JSON, reference arm, launch list, ncu full.
tag=${1:-full}
set -x
nproc > gpurun_out/nproc_$tag.txt; lscpu | head -20 > gpurun_out/lscpu_$tag.txt
nvidia-smi > gpurun_out/nvsmi_$tag.txt
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
# (the cfg4 scan sweep is part of bench.py now: its "lidar" section)
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 --no-lidar --no-replay > gpurun_out/plain_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 --no-lidar --no-replay > gpurun_out/ncu_launch_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:env_step_kernel -s 4 -c 1 -o gpurun_out/prof_step_$tag python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 --no-lidar --no-replay > gpurun_out/ncu_step_$tag.log 2>&1
echo done
