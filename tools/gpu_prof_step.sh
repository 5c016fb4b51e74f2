tag=${1:-pstep}
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 --no-lidar --no-replay > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:env_step_kernel -s 4 -c 1 -o gpurun_out/prof_step_$tag python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 --no-lidar --no-replay > gpurun_out/ncu_step_$tag.log 2>&1
echo rc=$?
