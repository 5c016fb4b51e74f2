# parity of the current build, then A/B: base (HEAD) vs current vs variants
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab4_tests.log
for lib in variants/lib_base.so default variants/lib_rs3.so variants/lib_t640.so; do
  if [ "$lib" = default ]; then unset SPARROW_LIB_PATH; else export SPARROW_LIB_PATH=$PWD/$lib; fi
  n=$(basename $lib)
  for b in 32 256; do timeout 120 python tools/bench_scan.py --beams $b > gpurun_out/ab4_${n}_$b.json 2>&1; done
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/ab4_${n}_bench.json 2>/dev/null
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/ab4_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "%.4f ms"%d.get("ms", d.get("ms_per_step", 0)))
    except Exception as e: print(f, open(f).read()[-300:])
PY
