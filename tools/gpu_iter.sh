# one GPU iteration: parity tests, N sweep, ncu of the step kernel (tag = $1)
tag=${1:-x}
set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_$tag.log
for n in 4096 65536 262144; do
  timeout 300 python bench.py --envs $n --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/scale_${tag}_$n.json 2>>gpurun_out/scale_$tag.err
done
if [ "${NCU:-1}" = "1" ]; then
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:env_step_kernel -s 3 -c 1 -o gpurun_out/prof_$tag python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ncu_$tag.log 2>&1
fi
cat gpurun_out/pytest_$tag.log
