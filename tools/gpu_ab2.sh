for lib in default variants/lib_scan1024.so; do
  if [ "$lib" = default ]; then unset SPARROW_LIB_PATH; else export SPARROW_LIB_PATH=$PWD/$lib; fi
  for b in 32 256; do timeout 120 python tools/bench_scan.py --beams $b > gpurun_out/ab2_$(basename $lib)_$b.json 2>&1; done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/ab2_*.json")):
    try: d=json.load(open(f)); print(f, "%.3f ms"%d["ms"], d["launch"])
    except Exception as e: print(f, open(f).read()[-300:])
PY
