for lib in variants/lib_timing.so variants/lib_timing_touch.so; do
  echo "== $lib"; SPARROW_LIB_PATH=$PWD/$lib timeout 300 python tools/debug/phase_ts.py 2>&1 | grep -v "^$"
done
for lib in default variants/lib_touch.so; do
  if [ "$lib" = default ]; then unset SPARROW_LIB_PATH; else export SPARROW_LIB_PATH=$PWD/$lib; fi
  echo "== $lib"
  timeout 300 python tools/debug/small_n.py 2>&1 | grep -E "flush "
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['ms_per_step'], d['value'])"
done
