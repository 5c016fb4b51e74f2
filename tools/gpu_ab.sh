# A/B: library variants x refill thresholds on the step bench (+ marcher)
for lib in default variants/lib_cta1.so; do
  for rm in 24 32 48; do
    if [ "$lib" = default ]; then unset SPARROW_LIB_PATH; else export SPARROW_LIB_PATH=$PWD/$lib; fi
    SPARROW_REFILL_MIN=$rm timeout 200 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ab_$(basename $lib)_$rm.json 2>/dev/null
    SPARROW_REFILL_MIN=$rm timeout 120 python tools/bench_scan.py > gpurun_out/abscan_$(basename $lib)_$rm.json 2>/dev/null
  done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/ab_*.json")):
    try:
        d=json.load(open(f)); s=json.load(open(f.replace("/ab_","/abscan_")))
        print(f, "step %.4f ms"%d["ms_per_step"], "median %.4f"%d["per_step_ms"]["median"], "scan %.3f ms"%s["ms"])
    except Exception as e: print(f, e)
PY
