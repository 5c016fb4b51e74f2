# quick iteration: gpu tests + marcher sweep (R=32/256 @300) + step bench
tag=${1:-q}
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4 > gpurun_out/pytest_$tag.log
for b in 32 256; do timeout 120 python tools/bench_scan.py --beams $b >> gpurun_out/scan_$tag.jsonl 2>>gpurun_out/scan_$tag.err; done
timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 5 > gpurun_out/step_$tag.json 2>>gpurun_out/step_$tag.err
cat gpurun_out/pytest_$tag.log
python - <<PY
import json
for l in open("gpurun_out/scan_$tag.jsonl"):
    d=json.loads(l); print("scan", d["beams"], "%.3f ms"%d["ms"], "%.3g rays/s"%d["rays_per_s"], "%.3g ray-cells/s"%d["ray_cells_per_s"])
d=json.load(open("gpurun_out/step_$tag.json")); print("step %.4f ms"%d["ms_per_step"], "%.3g env-steps/s"%d["value"], d["per_step_ms"], "e2e %.3g"%d["e2e"]["value"], d["clocks"])
PY
