for n in 4096 16384 65536 262144; do
  timeout 300 python bench.py --envs $n --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 5 > gpurun_out/sweep_$n.json 2>/dev/null
done
python - <<'PY'
import json
for n in (4096, 16384, 65536, 262144):
    try:
        d = json.load(open(f"gpurun_out/sweep_{n}.json"))
        print(n, "%.3e env-steps/s" % d["value"], "%.4f ms/step" % d["ms_per_step"], d["config"]["launch"])
    except Exception as e:
        print(n, "ERR", e)
PY
