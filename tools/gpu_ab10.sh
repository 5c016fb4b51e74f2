timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_ab10.log 2>&1; echo "rc=$?" >> gpurun_out/t_ab10.log
for lib in variants/lib_base4.so default variants/lib_base4.so default; do
  if [ "$lib" = default ]; then unset SPARROW_LIB_PATH; else export SPARROW_LIB_PATH=$PWD/$lib; fi
  echo "== $lib"
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['ms_per_step'], d['per_step_ms'])"
  timeout 300 python bench.py --envs 262144 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench256k', d['ms_per_step'])"
done
