set -x
for n in 4096 16384 65536 262144; do
  timeout 300 python bench.py --envs $n --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/scale_$n.json 2>>gpurun_out/scale.err
done
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:env_step_kernel -s 3 -c 1 -o gpurun_out/prof_step python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ncu.log 2>&1
echo done
