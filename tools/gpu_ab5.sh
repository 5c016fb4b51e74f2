for lib in default variants/lib_small.so; do
  if [ "$lib" = default ]; then unset SPARROW_LIB_PATH; else export SPARROW_LIB_PATH=$PWD/$lib; fi
  n=$(basename $lib)
  echo "== $n"
  timeout 300 python tools/debug/small_n.py 2>&1 | grep -E "b2b|flush " 
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['ms_per_step'], d['value'])"
done
