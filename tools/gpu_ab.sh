# A/B of library variants: step bench (65,536 envs) and the R=32 scan, interleaved.
# usage: bash tools/gpu_ab.sh TAG lib1.so lib2.so ...
tag=$1; shift
for rep in 1 2 3; do
  for lib in "$@"; do
    r=$(SPARROW_LIB_PATH=$lib timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f %.4f' % (d['ms_per_step'], d['per_step_ms']['median']))")
    s=$(SPARROW_LIB_PATH=$lib timeout 120 python tools/bench_scan.py --beams 32 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f' % d['ms'])")
    echo "$rep $lib step(mean,median) $r scan32 $s" | tee -a gpurun_out/ab_$tag.txt
  done
done
